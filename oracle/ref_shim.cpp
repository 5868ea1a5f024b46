// TEST INFRASTRUCTURE ONLY.  A C-callable shim over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/).  It is used by
// tests/golden/make_golden.py to produce golden vectors and by the CPU test-suite to cross-check the
// C restatement (oracle/specpar_oracle.c).  It is never linked into, or called by, the product.
//
// The only behavioural hook is the GNU-ld --wrap seam on specpar::forward_batch / specpar::forward
// (SURVEY.md Appendix A.3): TableModels registered here as "proxies" get their per-row distribution
// from a caller-supplied argmax callback (a one-hot row, so the reference's own argmax_token — strict
// '>' scan, lowest id on ties, model.cpp:70-81 — returns exactly the callback's id).  All other
// TableModels go to the real implementation.
#include <cstring>
#include <functional>
#include <optional>
#include <vector>
#include <map>
#include <mutex>
#include <sstream>
#include <string>

#include "specpar/datastore.hpp"
#include "specpar/harness.hpp"
#include "specpar/model.hpp"
#include "specpar/pipeline.hpp"
#include "specpar/verification.hpp"

using namespace specpar;

extern "C" {
typedef int (*ref_argmax_fn)(void* user, const int* ctx, int L, const int* cands, int c, int* out);
// full rows: out[(c+1) * vocab] fp64 next-token distributions
typedef int (*ref_probs_fn)(void* user, const int* ctx, int L, const int* cands, int c, double* out);
}

namespace {

struct Proxy {
    ref_argmax_fn fn;
    void* user;
    ref_probs_fn pfn = nullptr;  // when set, rows are the callback's distributions (sampled runs)
};
std::mutex g_mu;
std::map<const TableModel*, Proxy> g_proxies;

bool find_proxy(const TableModel* m, Proxy* out) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_proxies.find(m);
    if (it == g_proxies.end()) return false;
    *out = it->second;
    return true;
}

std::vector<ProbVector> proxy_rows(const TableModel& model, const Proxy& p,
                                   std::span<const TokenId> ctx, std::span<const TokenId> cands) {
    if (p.pfn) {
        const size_t V = static_cast<size_t>(model.vocab_size);
        std::vector<double> flat((cands.size() + 1) * V);
        if (p.pfn(p.user, ctx.data(), static_cast<int>(ctx.size()), cands.data(),
                  static_cast<int>(cands.size()), flat.data()) != 0) {
            throw std::runtime_error("proxy forward callback failed");
        }
        std::vector<ProbVector> rows;
        for (size_t r = 0; r <= cands.size(); ++r)
            rows.emplace_back(flat.begin() + static_cast<long>(r * V), flat.begin() + static_cast<long>((r + 1) * V));
        return rows;
    }
    std::vector<int> ids(cands.size() + 1);
    if (p.fn(p.user, ctx.data(), static_cast<int>(ctx.size()), cands.data(),
             static_cast<int>(cands.size()), ids.data()) != 0) {
        throw std::runtime_error("proxy forward callback failed");
    }
    std::vector<ProbVector> rows;
    rows.reserve(ids.size());
    for (int id : ids) {
        ProbVector r(static_cast<size_t>(model.vocab_size), 0.0);
        r[static_cast<size_t>(id)] = 1.0;
        rows.push_back(std::move(r));
    }
    return rows;
}

int copy_str(const std::string& s, char* buf, long cap) {
    if (!buf) return 0;
    if (static_cast<long>(s.size()) + 1 > cap) return -2;
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
    return 0;
}

void fill_metrics(const RunMetrics& m, double* out) {
    if (!out) return;
    out[0] = static_cast<double>(m.tokens);
    out[1] = static_cast<double>(m.rounds);
    out[2] = m.clock;
    out[3] = m.m;
    out[4] = m.amt;
    out[5] = m.speedup;
    out[6] = m.hit_rate;
    out[7] = static_cast<double>(m.lookups);
}

thread_local std::string g_err;

}  // namespace

// ---- the link seam -------------------------------------------------------------------------
// C linkage so the symbols are literally __wrap_<mangled> / __real_<mangled>.
extern "C" {
std::vector<ProbVector> __real__ZN7specpar13forward_batchERKNS_10TableModelESt4spanIKiLm18446744073709551615EES5_PNS_8SimClockE(
    const TableModel&, std::span<const TokenId>, std::span<const TokenId>, SimClock*);
ProbVector __real__ZN7specpar7forwardERKNS_10TableModelESt4spanIKiLm18446744073709551615EEPNS_8SimClockE(
    const TableModel&, std::span<const TokenId>, SimClock*);

std::vector<ProbVector> __wrap__ZN7specpar13forward_batchERKNS_10TableModelESt4spanIKiLm18446744073709551615EES5_PNS_8SimClockE(
    const TableModel& model, std::span<const TokenId> ctx, std::span<const TokenId> cands,
    SimClock* clock) {
    Proxy p;
    if (!find_proxy(&model, &p)) {
        return __real__ZN7specpar13forward_batchERKNS_10TableModelESt4spanIKiLm18446744073709551615EES5_PNS_8SimClockE(
            model, ctx, cands, clock);
    }
    if (ctx.empty()) throw std::invalid_argument("forward_batch: empty context");
    if (clock) clock->charge(model.forward_cost);
    return proxy_rows(model, p, ctx, cands);
}

ProbVector __wrap__ZN7specpar7forwardERKNS_10TableModelESt4spanIKiLm18446744073709551615EEPNS_8SimClockE(
    const TableModel& model, std::span<const TokenId> ctx, SimClock* clock) {
    Proxy p;
    if (!find_proxy(&model, &p)) {
        return __real__ZN7specpar7forwardERKNS_10TableModelESt4spanIKiLm18446744073709551615EEPNS_8SimClockE(
            model, ctx, clock);
    }
    if (ctx.empty()) throw std::invalid_argument("forward: empty context");
    if (clock) clock->charge(model.forward_cost);
    return proxy_rows(model, p, ctx, {}).front();
}
}  // extern "C" (link seam)

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Runs method `method` on the key=value config `cfg_text` exactly as the reference harness does
// (run_method_on, harness.cpp:403-429).  metrics[8] = tokens, rounds, clock, m, amt, speedup,
// hit_rate, lookups.
int ref_run_config(const char* cfg_text, const char* method, int* out_tokens, int cap, int* n_out,
                   char* jsonl, long jsonl_cap, double* metrics) {
    try {
        const ExperimentConfig cfg = parse_config(cfg_text);
        const ExperimentSetup setup = build_setup(cfg);
        RunResult res;
        run_method_on(cfg, setup, parse_method(method), &res);
        if (static_cast<int>(res.output.size()) > cap) return -2;
        std::memcpy(out_tokens, res.output.data(), res.output.size() * sizeof(int));
        *n_out = static_cast<int>(res.output.size());
        fill_metrics(res.metrics, metrics);
        return copy_str(traces_to_jsonl(res.traces), jsonl, jsonl_cap);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Exports the deterministic setup of a config: model-v1 texts, dstore-v1 prior, prompt.
int ref_export_setup(const char* cfg_text, char* draft_buf, long draft_cap, char* target_buf,
                     long target_cap, char* prior_buf, long prior_cap, int* prompt, int* n_prompt,
                     int prompt_cap) {
    try {
        const ExperimentConfig cfg = parse_config(cfg_text);
        const ExperimentSetup setup = build_setup(cfg);
        const HierarchicalDatastore store = build_store(cfg, setup.corpus);
        if (static_cast<int>(setup.prompt.size()) > prompt_cap) return -2;
        std::memcpy(prompt, setup.prompt.data(), setup.prompt.size() * sizeof(int));
        *n_prompt = static_cast<int>(setup.prompt.size());
        int rc = copy_str(serialize_model(setup.draft_model), draft_buf, draft_cap);
        if (rc) return rc;
        rc = copy_str(serialize_model(setup.target_model), target_buf, target_cap);
        if (rc) return rc;
        return copy_str(serialize_index(store.prior), prior_buf, prior_cap);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// gen_corpus (harness.cpp:151-186) flattened: out_tokens gets the concatenation, seq_lens the split.
int ref_gen_corpus(int vocab, double rho, int length, unsigned long long seed, int* out_tokens,
                   int* seq_lens, int* n_seqs, int seq_cap) {
    try {
        const auto corpus = gen_corpus(vocab, rho, length, seed);
        if (static_cast<int>(corpus.size()) > seq_cap) return -2;
        int at = 0;
        for (size_t i = 0; i < corpus.size(); ++i) {
            std::memcpy(out_tokens + at, corpus[i].data(), corpus[i].size() * sizeof(int));
            at += static_cast<int>(corpus[i].size());
            seq_lens[i] = static_cast<int>(corpus[i].size());
        }
        *n_seqs = static_cast<int>(corpus.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// A HierarchicalDatastore built from explicit (layer, tokens, step) inserts, then a batch of lookups
// on the same store (stats accumulate).  layer: 0 prior, 1 dynamic, 2 rejected.
// Per lookup q: out_n[q], out_source[q] (LookupSource enum order), out_order[q], and candidates in
// out_cands[q*d_cap ...].  stats[6] = lookups, prior, dynamic, rejected, fallback, misses.
int ref_lookup_batch(int max_order, int depth_cfg, int rejected_enabled, int n_ins,
                     const int* ins_layer, const int* ins_len, const long* ins_step,
                     const int* ins_tokens, int n_q, const int* q_len, const int* q_tokens,
                     const int* q_depth, int d_cap, int* out_cands, int* out_n, int* out_source,
                     int* out_order, long* stats) {
    try {
        HierarchicalDatastore store(max_order, depth_cfg);
        store.rejected_enabled = rejected_enabled != 0;
        int at = 0;
        for (int i = 0; i < n_ins; ++i) {
            std::span<const TokenId> toks(ins_tokens + at, static_cast<size_t>(ins_len[i]));
            NGramIndex* layer = ins_layer[i] == 0 ? &store.prior
                                : ins_layer[i] == 1 ? &store.dynamic : &store.rejected;
            layer->insert(toks, ins_step[i]);
            at += ins_len[i];
        }
        at = 0;
        for (int q = 0; q < n_q; ++q) {
            std::span<const TokenId> ctx(q_tokens + at, static_cast<size_t>(q_len[q]));
            at += q_len[q];
            const LookupResult r = store.lookup(ctx, q_depth[q]);
            if (static_cast<int>(r.candidates.size()) > d_cap) return -2;
            std::memcpy(out_cands + static_cast<long>(q) * d_cap, r.candidates.data(),
                        r.candidates.size() * sizeof(int));
            out_n[q] = static_cast<int>(r.candidates.size());
            out_source[q] = static_cast<int>(r.source);
            out_order[q] = r.matched_order;
        }
        stats[0] = store.stats.lookups.load();
        stats[1] = store.stats.prior_hits.load();
        stats[2] = store.stats.dynamic_hits.load();
        stats[3] = store.stats.rejected_hits.load();
        stats[4] = store.stats.fallback_hits.load();
        stats[5] = store.stats.misses.load();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The reference decode loop run() (pipeline.cpp:264-323) with callback-backed proxy models.
// prior: n_prior sequences (steps 0..n_prior-1 as build_prior assigns, datastore.cpp:149-159).
// Greedy only (temperature 0).  metrics as in ref_run_config.
int ref_run_callback(int vocab, ref_argmax_fn draft_fn, void* draft_user, ref_argmax_fn target_fn,
                     void* target_user, int max_order, int n_prior, const int* prior_lens,
                     const int* prior_tokens, const int* prompt, int n_prompt, int max_new,
                     int gamma, int depth, int draft_retrieval, int target_retrieval,
                     int rejected_enabled, double t_target, double t_draft, double t_lookup,
                     double t_sync, int* out_tokens, int cap, int* n_out, char* jsonl,
                     long jsonl_cap, double* metrics) {
    TableModel draft, target;
    draft.vocab_size = target.vocab_size = vocab;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_proxies[&draft] = {draft_fn, draft_user};
        g_proxies[&target] = {target_fn, target_user};
    }
    int rc = 0;
    try {
        HierarchicalDatastore store(max_order, depth);
        store.prior.max_order = max_order;
        int at = 0;
        for (int i = 0; i < n_prior; ++i) {
            store.prior.insert(std::span<const TokenId>(prior_tokens + at,
                                                        static_cast<size_t>(prior_lens[i])),
                               i);
            at += prior_lens[i];
        }
        store.rejected_enabled = rejected_enabled != 0;
        PipelineOptions opts;
        opts.gamma = gamma;
        opts.depth = depth;
        opts.draft_retrieval = draft_retrieval != 0;
        opts.target_retrieval = target_retrieval != 0;
        opts.latency = {t_target, t_draft, t_lookup, t_sync};
        const TokenSeq p(prompt, prompt + n_prompt);
        const RunResult res = run(draft, target, store, p, max_new, opts);
        if (static_cast<int>(res.output.size()) > cap) {
            rc = -2;
        } else {
            std::memcpy(out_tokens, res.output.data(), res.output.size() * sizeof(int));
            *n_out = static_cast<int>(res.output.size());
            fill_metrics(res.metrics, metrics);
            rc = copy_str(traces_to_jsonl(res.traces), jsonl, jsonl_cap);
        }
    } catch (const std::exception& e) {
        g_err = e.what();
        rc = -1;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_proxies.erase(&draft);
    g_proxies.erase(&target);
    return rc;
}

}  // extern "C"

// ---- verifier (verification.cpp:19-132) over the unmodified reference; a Rng handle per stream
namespace {
std::vector<ProbVector> rows_of(const double* data, const long* off, int n) {
    std::vector<ProbVector> r;
    for (int i = 0; i < n; ++i) r.emplace_back(data + off[i], data + off[i + 1]);
    return r;
}
int ref_guard(const std::function<void()>& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}
}  // namespace

extern "C" {
void* ref_rng_new(unsigned long long seed) { return new Rng(seed); }
void* ref_rng_derive(unsigned long long seed, unsigned long long round, unsigned long long lane) {
    return new Rng(derive_rng(seed, round, lane));
}
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
double ref_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
int ref_accept_prob(const double* p, int np, const double* q, int nq, int x, double* out) {
    return ref_guard([&] { *out = accept_prob(ProbVector(p, p + np), ProbVector(q, q + nq), x); });
}
int ref_residual_sample(const double* p, int np, const double* q, int nq, void* rng, int* out) {
    return ref_guard([&] { *out = residual_sample(ProbVector(p, p + np), ProbVector(q, q + nq), *static_cast<Rng*>(rng)); });
}
int ref_residual_point_mass(const double* p, int np, int x, void* rng, int* out) {
    return ref_guard([&] { *out = residual_sample_point_mass(ProbVector(p, p + np), x, *static_cast<Rng*>(rng)); });
}
int ref_verify_against_target(const int* draft, int n_draft, const double* dp, const long* doff, int n_dp,
                              const double* tp, const long* toff, int n_tp, double temperature, void* rng,
                              int* first_reject) {
    return ref_guard([&] {
        const std::vector<ProbVector> d = rows_of(dp, doff, n_dp), t = rows_of(tp, toff, n_tp);
        const std::vector<TokenId> dt(draft, draft + n_draft);
        SamplerConfig cfg{temperature, 0};
        const std::optional<int> r = verify_against_target(dt, d, t, cfg, *static_cast<Rng*>(rng));
        *first_reject = r ? *r : -1;
    });
}
int ref_guided_output(const int* draft, int n_draft, const double* dp, const long* doff, int n_dp, const int* gtok,
                      int n_gtok, const double* gp, const long* goff, int n_gp, int first_reject, double temperature,
                      void* rng, int* committed, int cap, int* n_committed, int* accepted_len, int* kind) {
    return ref_guard([&] {
        const std::vector<ProbVector> d = rows_of(dp, doff, n_dp);
        GuidanceChain g;
        g.tokens.assign(gtok, gtok + n_gtok);
        g.probs = rows_of(gp, goff, n_gp);
        const std::vector<TokenId> dt(draft, draft + n_draft);
        SamplerConfig cfg{temperature, 0};
        const std::optional<int> fr = first_reject < 0 ? std::nullopt : std::optional<int>(first_reject);
        const VerifyOutcome o = guided_output(dt, d, g, fr, cfg, *static_cast<Rng*>(rng));
        *n_committed = static_cast<int>(o.committed.size());
        *accepted_len = o.accepted_len;
        *kind = static_cast<int>(o.kind);
        for (int i = 0; i < *n_committed && i < cap; ++i) committed[i] = o.committed[static_cast<size_t>(i)];
    });
}
// The same loop at temperature > 0: proxy models return full fp64 rows from the callbacks and the
// reference's own accept_with_model / finish_round / derive_rng run unmodified (SamplerConfig
// {temperature, seed}).  method "double" = run() with the given retrieval flags; "vanilla_ar", "sd",
// "draft_retrieval" = the harness entry points (harness.cpp:233-369) through run_method_on, with the
// prior rebuilt by build_store from the same sequences.
int ref_run_callback_probs(int vocab, ref_probs_fn draft_fn, void* draft_user, ref_probs_fn target_fn,
                           void* target_user, int max_order, int n_prior, const int* prior_lens,
                           const int* prior_tokens, const int* prompt, int n_prompt, int max_new, int gamma,
                           int depth, int draft_retrieval, int target_retrieval, int rejected_enabled,
                           double t_target, double t_draft, double t_lookup, double t_sync, double temperature,
                           unsigned long long seed, const char* method, int* out_tokens, int cap, int* n_out,
                           char* jsonl, long jsonl_cap, double* metrics) {
    ExperimentSetup setup;
    setup.draft_model.vocab_size = setup.target_model.vocab_size = vocab;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        g_proxies[&setup.draft_model] = {nullptr, draft_user, draft_fn};
        g_proxies[&setup.target_model] = {nullptr, target_user, target_fn};
    }
    int rc = 0;
    try {
        setup.prompt.assign(prompt, prompt + n_prompt);
        int at = 0;
        for (int i = 0; i < n_prior; ++i) {
            setup.corpus.emplace_back(prior_tokens + at, prior_tokens + at + prior_lens[i]);
            at += prior_lens[i];
        }
        RunResult res;
        if (std::string(method) == "double") {
            HierarchicalDatastore store(max_order, depth);
            store.prior.max_order = max_order;
            for (int i = 0; i < n_prior; ++i) store.prior.insert(setup.corpus[static_cast<size_t>(i)], i);
            store.rejected_enabled = rejected_enabled != 0;
            PipelineOptions opts;
            opts.gamma = gamma;
            opts.depth = depth;
            opts.draft_retrieval = draft_retrieval != 0;
            opts.target_retrieval = target_retrieval != 0;
            opts.latency = {t_target, t_draft, t_lookup, t_sync};
            opts.sampler = SamplerConfig{temperature, seed};
            res = run(setup.draft_model, setup.target_model, store, setup.prompt, max_new, opts);
        } else {
            ExperimentConfig cfg;
            cfg.vocab = vocab;
            cfg.gamma = gamma;
            cfg.depth = depth;
            cfg.ngram = max_order;
            cfg.prior_rounds = n_prior;
            cfg.rejected_cache = rejected_enabled != 0;
            cfg.latency = {t_target, t_draft, t_lookup, t_sync};
            cfg.temperature = temperature;
            cfg.seed = seed;
            cfg.max_new_tokens = max_new;
            run_method_on(cfg, setup, parse_method(method), &res);
        }
        if (static_cast<int>(res.output.size()) > cap) {
            rc = -2;
        } else {
            std::memcpy(out_tokens, res.output.data(), res.output.size() * sizeof(int));
            *n_out = static_cast<int>(res.output.size());
            fill_metrics(res.metrics, metrics);
            rc = copy_str(traces_to_jsonl(res.traces), jsonl, jsonl_cap);
        }
    } catch (const std::exception& e) {
        g_err = e.what();
        rc = -1;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_proxies.erase(&setup.draft_model);
    g_proxies.erase(&setup.target_model);
    return rc;
}

}  // extern "C"
