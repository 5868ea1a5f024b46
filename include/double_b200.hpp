// double_b200.hpp — header-only C++ mirror of the reference's decode-path API
// (/root/reference/proj/include/specpar/*.hpp) over the C-ABI in double_b200.h.
//
// A C++ caller of specpar::HierarchicalDatastore / forward_batch / run switches to the same names in
// namespace specpar_b200; errors surface as the reference's exception types
// (std::invalid_argument, std::runtime_error, std::logic_error — pipeline.cpp:18-22, 210-217).
#pragma once
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "double_b200.h"

namespace specpar_b200 {

using TokenId = std::int32_t;       // types.hpp:10
using TokenSeq = std::vector<TokenId>;

inline void check(int status) {
    if (status == DBL_OK) return;
    const std::string msg = dbl_last_error();
    switch (status) {
        case DBL_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case DBL_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

enum class LookupSource { Prior, Dynamic, Rejected, ContextFallback, Miss };  // datastore.hpp:29

struct LookupResult {  // datastore.hpp:33-37
    TokenSeq candidates;
    LookupSource source = LookupSource::Miss;
    int matched_order = 0;
};

struct LookupStats {  // datastore.hpp:39-67 (a snapshot of the device counters)
    long lookups = 0, prior_hits = 0, dynamic_hits = 0, rejected_hits = 0, fallback_hits = 0, misses = 0;
    long hits() const { return prior_hits + dynamic_hits + rejected_hits + fallback_hits; }
    double hit_rate() const { return lookups == 0 ? 0.0 : static_cast<double>(hits()) / lookups; }
};

class HierarchicalDatastore;

class NGramIndex {  // one device layer (datastore.hpp:19-27)
  public:
    void insert(std::span<const TokenId> tokens, long step);
    size_t occurrence_count() const;
    void clear();

  private:
    friend class HierarchicalDatastore;
    NGramIndex(HierarchicalDatastore* s, int layer) : s_(s), layer_(layer) {}
    HierarchicalDatastore* s_;
    int layer_;
};

class HierarchicalDatastore {  // datastore.hpp:72-95
  public:
    explicit HierarchicalDatastore(int n = 3, int d = 10, int device = 0) : max_order(n), depth(d) {
        check(dbl_store_create(n, d, device, &h_));
    }
    ~HierarchicalDatastore() { dbl_store_destroy(h_); }
    HierarchicalDatastore(const HierarchicalDatastore&) = delete;
    HierarchicalDatastore& operator=(const HierarchicalDatastore&) = delete;

    NGramIndex prior{this, DBL_LAYER_PRIOR}, dynamic{this, DBL_LAYER_DYNAMIC}, rejected{this, DBL_LAYER_REJECTED};
    int max_order, depth;

    void set_rejected_enabled(bool on) { check(dbl_store_set_rejected_enabled(h_, on ? 1 : 0)); }
    LookupResult lookup(std::span<const TokenId> context, int d) const {  // datastore.cpp:82-132
        LookupResult r;
        r.candidates.resize(static_cast<size_t>(d > 0 ? d : 1));
        int n = 0, src = 0, order = 0;
        check(dbl_store_lookup(h_, context.data(), static_cast<int>(context.size()), d, r.candidates.data(),
                               static_cast<int>(r.candidates.size()), &n, &src, &order));
        r.candidates.resize(static_cast<size_t>(n));
        r.source = static_cast<LookupSource>(src);
        r.matched_order = order;
        return r;
    }
    void record_accepted(std::span<const TokenId> t) {  // datastore.cpp:134-137
        check(dbl_store_record(h_, DBL_LAYER_DYNAMIC, t.data(), static_cast<int>(t.size())));
    }
    void record_rejected(std::span<const TokenId> t) {  // datastore.cpp:139-142
        check(dbl_store_record(h_, DBL_LAYER_REJECTED, t.data(), static_cast<int>(t.size())));
    }
    void flush_session() { check(dbl_store_flush_session(h_)); }  // datastore.cpp:144-147
    LookupStats stats() const {
        int64_t v[6];
        check(dbl_store_stats(h_, v));
        return {v[0], v[1], v[2], v[3], v[4], v[5]};
    }
    dbl_store_t handle() const { return h_; }

  private:
    dbl_store_t h_ = nullptr;
};

inline void NGramIndex::insert(std::span<const TokenId> tokens, long step) {  // datastore.cpp:9-20
    check(dbl_store_insert(s_->handle(), layer_, tokens.data(), static_cast<int>(tokens.size()), step));
}
inline size_t NGramIndex::occurrence_count() const {  // datastore.cpp:22-26
    int64_t ns = 0, nt = 0, occ = 0;
    check(dbl_store_layer_info(s_->handle(), layer_, &ns, &nt, &occ));
    return static_cast<size_t>(occ);
}
inline void NGramIndex::clear() { check(dbl_store_clear_layer(s_->handle(), layer_)); }

// build_prior (datastore.cpp:149-159): the first K sequences, step = index, into store.prior
inline void build_prior(HierarchicalDatastore& store, const std::vector<TokenSeq>& corpora, int rounds) {
    if (rounds < 0) throw std::invalid_argument("build_prior: rounds must be >= 0");
    for (size_t i = 0; i < corpora.size() && static_cast<int>(i) < rounds; ++i)
        store.prior.insert(corpora[i], static_cast<long>(i));
}

class Model {  // TableModel / transformer behind forward_batch (model.hpp:18-48)
  public:
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;
    Model(Model&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~Model() { if (h_) dbl_model_destroy(h_); }
    int vocab_size() const {
        int v = 0;
        check(dbl_model_vocab(h_, &v));
        return v;
    }
    dbl_model_t handle() const { return h_; }
    static Model table(int order, int vocab, const std::vector<int32_t>& windows, const std::vector<double>& probs,
                       const std::vector<double>& fallback, int device = 0) {
        dbl_model_t h = nullptr;
        check(dbl_table_create(order, vocab, static_cast<int64_t>(windows.size() / order), windows.data(), probs.data(),
                               fallback.data(), device, &h));
        return Model(h);
    }
    static Model transformer(const dbl_transformer_config& cfg, int device = 0) {
        dbl_model_t h = nullptr;
        check(dbl_transformer_create(&cfg, device, nullptr, &h));
        return Model(h);
    }

  private:
    explicit Model(dbl_model_t h) : h_(h) {}
    dbl_model_t h_ = nullptr;
};

// forward_batch (model.cpp:37-53) consumed greedily: argmax_token of each of the |cands|+1 rows
inline TokenSeq forward_batch_argmax(const Model& m, std::span<const TokenId> ctx, std::span<const TokenId> cands) {
    TokenSeq out(cands.size() + 1);
    check(dbl_forward_argmax(m.handle(), ctx.data(), static_cast<int>(ctx.size()), cands.data(),
                             static_cast<int>(cands.size()), out.data()));
    return out;
}

struct SamplerConfig {  // model.hpp:11-14
    double temperature = 0.0;
    std::uint64_t rng_seed = 0;
};

struct PipelineOptions {  // pipeline.hpp:36-44 (+ LatencyConfig :15-29)
    int gamma = 4, depth = 10;
    bool draft_retrieval = true, target_retrieval = true;
    double t_target = 1.0, t_draft = 0.25, t_lookup = 0.0, t_sync = 0.0;
    SamplerConfig sampler{};
};

struct RunResult {  // pipeline.hpp:84-88 (traces as the traces_to_jsonl text)
    TokenSeq output;
    dbl_run_metrics metrics{};
    std::string jsonl;
};

namespace detail {
inline dbl_pipeline_options c_options(const PipelineOptions& o) {
    return dbl_pipeline_options{o.gamma, o.depth, o.draft_retrieval, o.target_retrieval, 1,
                                o.t_target, o.t_draft, o.t_lookup, o.t_sync, 1, o.sampler.temperature,
                                o.sampler.rng_seed};
}
inline void flatten(const std::vector<TokenSeq>& seqs, std::vector<int64_t>& off, TokenSeq& flat) {
    off.assign(1, 0);
    flat.clear();
    for (const TokenSeq& s : seqs) {
        flat.insert(flat.end(), s.begin(), s.end());
        off.push_back(static_cast<int64_t>(flat.size()));
    }
    if (flat.empty()) flat.push_back(0);
}
}  // namespace detail

// run (pipeline.cpp:264-323)
inline RunResult run(const Model& draft, const Model& target, HierarchicalDatastore& store, const TokenSeq& prompt,
                     int max_new_tokens, const PipelineOptions& o) {
    const dbl_pipeline_options c = detail::c_options(o);
    RunResult r;
    r.output.resize(static_cast<size_t>(max_new_tokens > 0 ? max_new_tokens : 1));
    int n = 0;
    int64_t jl = 0;
    check(dbl_run(draft.handle(), target.handle(), store.handle(), prompt.data(), static_cast<int>(prompt.size()),
                  max_new_tokens, &c, r.output.data(), static_cast<int>(r.output.size()), &n, &r.metrics, nullptr, 0, &jl));
    r.output.resize(static_cast<size_t>(n));
    (void)jl;
    return r;
}


// Batched DOUBLE: run() for several sequences, one datastore each, sharing every
// forward; result b == run(draft, target, *stores[b], prompts[b], ...) alone.
inline std::vector<RunResult> run_batch(const Model& draft, const Model& target,
                                        const std::vector<HierarchicalDatastore*>& stores,
                                        const std::vector<TokenSeq>& prompts, int max_new_tokens,
                                        const PipelineOptions& o) {
    const dbl_pipeline_options c = detail::c_options(o);
    std::vector<int64_t> off;
    TokenSeq flat;
    detail::flatten(prompts, off, flat);
    const int B = static_cast<int>(prompts.size()), n = max_new_tokens > 0 ? max_new_tokens : 1;
    std::vector<dbl_store_t> hs;
    for (HierarchicalDatastore* st : stores) hs.push_back(st->handle());
    TokenSeq out(static_cast<size_t>(B) * n);
    std::vector<int32_t> out_n(static_cast<size_t>(B > 0 ? B : 1));
    std::vector<dbl_run_metrics> m(static_cast<size_t>(B > 0 ? B : 1));
    check(dbl_run_batch(draft.handle(), target.handle(), B, hs.data(), off.data(), flat.data(), max_new_tokens, &c,
                        out.data(), out_n.data(), m.data(), nullptr, 0, nullptr));
    std::vector<RunResult> rs(static_cast<size_t>(B));
    for (int b = 0; b < B; ++b) {
        rs[b].output.assign(out.begin() + static_cast<long>(b) * n, out.begin() + static_cast<long>(b) * n + out_n[b]);
        rs[b].metrics = m[b];
    }
    return rs;
}

// Batched serving: run_vanilla_ar for several prompts in lockstep, one forward per step over all
inline std::vector<TokenSeq> run_vanilla_ar_batch(const Model& target, const std::vector<TokenSeq>& prompts,
                                                  int max_new_tokens, double* device_ms = nullptr) {
    std::vector<int64_t> off;
    TokenSeq flat;
    detail::flatten(prompts, off, flat);
    const int B = static_cast<int>(prompts.size()), n = max_new_tokens > 0 ? max_new_tokens : 1;
    TokenSeq out(static_cast<size_t>(B) * n);
    std::vector<int32_t> out_n(static_cast<size_t>(B > 0 ? B : 1));
    double ms = 0.0;
    int64_t launches = 0;
    check(dbl_run_ar_batch(target.handle(), B, off.data(), flat.data(), max_new_tokens, out.data(), out_n.data(), &ms,
                           &launches));
    if (device_ms) *device_ms = ms;
    std::vector<TokenSeq> rs(static_cast<size_t>(B));
    for (int b = 0; b < B; ++b)
        rs[b].assign(out.begin() + static_cast<long>(b) * n, out.begin() + static_cast<long>(b) * n + out_n[b]);
    return rs;
}

// forward_batch (model.cpp:37-53) as ProbVector rows: (|cands|+1) x vocab fp64
inline std::vector<std::vector<double>> forward_batch(const Model& m, std::span<const TokenId> ctx,
                                                      std::span<const TokenId> cands) {
    const int V = m.vocab_size();
    std::vector<double> flat((cands.size() + 1) * static_cast<size_t>(V));
    check(dbl_forward_dists(m.handle(), ctx.data(), static_cast<int>(ctx.size()), cands.data(),
                            static_cast<int>(cands.size()), flat.data()));
    std::vector<std::vector<double>> rows;
    for (size_t r = 0; r <= cands.size(); ++r)
        rows.emplace_back(flat.begin() + static_cast<long>(r * V), flat.begin() + static_cast<long>((r + 1) * V));
    return rows;
}

// run_vanilla_ar (harness.cpp:233-258)
inline RunResult run_vanilla_ar(const Model& target, const TokenSeq& prompt, int max_new_tokens, double t_target = 1.0,
                                const SamplerConfig& sampler = {}) {
    RunResult r;
    r.output.resize(static_cast<size_t>(max_new_tokens > 0 ? max_new_tokens : 1));
    int n = 0;
    int64_t jl = 0;
    check(dbl_run_ar_sampled(target.handle(), prompt.data(), static_cast<int>(prompt.size()), max_new_tokens,
                             t_target, sampler.temperature, sampler.rng_seed, r.output.data(),
                             static_cast<int>(r.output.size()), &n, &r.metrics, nullptr, 0, &jl));
    r.output.resize(static_cast<size_t>(n));
    return r;
}

// ------------------------------------------------------------------ verifier + RNG (verification.hpp, rng.hpp)
using ProbVector = std::vector<double>;  // types.hpp

class Rng {  // rng.hpp:19-30 — the mt19937_64 stream lives on the device
  public:
    explicit Rng(std::uint64_t seed, int device = 0) { check(dbl_rng_create(seed, device, &h_)); }
    Rng(const Rng&) = delete;
    Rng& operator=(const Rng&) = delete;
    Rng(Rng&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~Rng() { if (h_) dbl_rng_destroy(h_); }
    double uniform() {
        double u = 0.0;
        check(dbl_rng_uniform(h_, &u, 1));
        return u;
    }
    dbl_rng_t handle() const { return h_; }
    static Rng derived(std::uint64_t seed, std::uint64_t round, std::uint64_t lane, int device = 0) {
        dbl_rng_t h = nullptr;
        check(dbl_rng_derive(seed, round, lane, device, &h));
        return Rng(h);
    }

  private:
    explicit Rng(dbl_rng_t h) : h_(h) {}
    dbl_rng_t h_ = nullptr;
};
inline Rng derive_rng(std::uint64_t seed, std::uint64_t round, std::uint64_t lane) {  // rng.hpp:33-35
    return Rng::derived(seed, round, lane);
}

struct GuidanceChain {  // verification.hpp:13-17
    TokenSeq tokens;
    std::vector<ProbVector> probs;
    int matched_len = 0;
};
enum class VerifyKind { AllAccepted, Correction, Extension, ResidualCorrection };  // verification.hpp:20
struct VerifyOutcome {  // verification.hpp:22-26
    int accepted_len = 0;
    TokenSeq committed;
    VerifyKind kind = VerifyKind::AllAccepted;
};

namespace detail {
struct Rows {  // ragged rows -> flat + offsets
    std::vector<double> data;
    std::vector<std::int64_t> off{0};
    explicit Rows(std::span<const ProbVector> rows) {
        for (const auto& r : rows) {
            data.insert(data.end(), r.begin(), r.end());
            off.push_back(static_cast<std::int64_t>(data.size()));
        }
        if (data.empty()) data.push_back(0.0);
    }
    int n() const { return static_cast<int>(off.size()) - 1; }
};
}  // namespace detail

inline double accept_prob(const ProbVector& p, const ProbVector& q, TokenId x) {  // verification.cpp:19-23
    double out = 0.0;
    check(dbl_accept_prob(p.data(), static_cast<int>(p.size()), q.data(), static_cast<int>(q.size()), x, &out));
    return out;
}
inline TokenId residual_sample(const ProbVector& p, const ProbVector& q, Rng& rng) {  // :40-50
    TokenId out = -1;
    check(dbl_residual_sample(p.data(), static_cast<int>(p.size()), q.data(), static_cast<int>(q.size()),
                              rng.handle(), &out));
    return out;
}
inline TokenId residual_sample_point_mass(const ProbVector& p, TokenId x, Rng& rng) {  // :52-58
    TokenId out = -1;
    check(dbl_residual_sample_point_mass(p.data(), static_cast<int>(p.size()), x, rng.handle(), &out));
    return out;
}
inline std::optional<int> verify_against_target(std::span<const TokenId> draft_tokens,
                                                std::span<const ProbVector> draft_probs,
                                                std::span<const ProbVector> target_probs, const SamplerConfig& cfg,
                                                Rng& rng) {  // verification.cpp:60-78
    const detail::Rows d(draft_probs), t(target_probs);
    int fr = -1;
    check(dbl_verify_against_target(draft_tokens.data(), static_cast<int>(draft_tokens.size()), d.data.data(),
                                    d.off.data(), d.n(), t.data.data(), t.off.data(), t.n(), cfg.temperature,
                                    rng.handle(), &fr));
    return fr < 0 ? std::nullopt : std::optional<int>(fr);
}
inline VerifyOutcome guided_output(std::span<const TokenId> draft_tokens, std::span<const ProbVector> draft_probs,
                                   const GuidanceChain& guidance, std::optional<int> first_reject,
                                   const SamplerConfig& cfg, Rng& rng) {  // verification.cpp:80-132
    const detail::Rows d(draft_probs), g(guidance.probs);
    TokenSeq out(draft_tokens.size() + guidance.tokens.size() + 1);
    int n = 0, acc = 0, kind = 0;
    check(dbl_guided_output(draft_tokens.data(), static_cast<int>(draft_tokens.size()), d.data.data(), d.off.data(),
                            d.n(), guidance.tokens.data(), static_cast<int>(guidance.tokens.size()), g.data.data(),
                            g.off.data(), g.n(), first_reject ? *first_reject : -1, cfg.temperature, rng.handle(),
                            out.data(), static_cast<int>(out.size()), &n, &acc, &kind));
    out.resize(static_cast<size_t>(n));
    return VerifyOutcome{acc, out, static_cast<VerifyKind>(kind)};
}

}  // namespace specpar_b200
