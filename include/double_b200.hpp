// double_b200.hpp — header-only C++ mirror of the reference's decode-path API
// (/root/reference/proj/include/specpar/*.hpp) over the C-ABI in double_b200.h.
//
// A C++ caller of specpar::HierarchicalDatastore / forward_batch / run switches to the same names in
// namespace specpar_b200; errors surface as the reference's exception types
// (std::invalid_argument, std::runtime_error, std::logic_error — pipeline.cpp:18-22, 210-217).
#pragma once
#include <cstdint>
#include <cstring>
#include <memory>
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

// NGramIndex (datastore.hpp:19-27).  Two faces: a host VALUE (what build_prior / parse_index return in
// the reference: max_order + the stored sequences) and a store LAYER (store.prior/dynamic/rejected, in
// HBM).  Assigning a value to a layer loads it onto the device in one upload; lookups run on the device.
class NGramIndex {
  public:
    NGramIndex() = default;
    NGramIndex(const NGramIndex& o) : max_order(o.max_order), sequences(o.materialize()), steps_(o.steps()) {}
    NGramIndex& operator=(const NGramIndex& o);
    int max_order = 3;
    std::vector<TokenSeq> sequences;  // the value face (a layer's are read back by materialize())

    void insert(std::span<const TokenId> tokens, long step);
    size_t occurrence_count() const;
    void clear();
    bool is_layer() const { return s_ != nullptr; }
    std::vector<TokenSeq> materialize() const;  // the stored sequences (copied back from HBM for a layer)
    std::vector<long> steps() const;

  private:
    friend class HierarchicalDatastore;
    NGramIndex(HierarchicalDatastore* s, int layer) : s_(s), layer_(layer) {}
    HierarchicalDatastore* s_ = nullptr;
    int layer_ = -1;
    std::vector<long> steps_;
};

class HierarchicalDatastore {  // datastore.hpp:72-95
  public:
    explicit HierarchicalDatastore(int n = 3, int d = 10, int device = 0) : max_order(n), depth(d) {
        check(dbl_store_create(n, d, device, &h_));
    }
    ~HierarchicalDatastore() { if (h_) dbl_store_destroy(h_); }
    // the reference's store is a value type (test_pipeline.cpp:170-187): copies are deep, on the device
    HierarchicalDatastore(const HierarchicalDatastore& o) : max_order(o.max_order), depth(o.depth) {
        check(dbl_store_clone(o.h_, &h_));
    }
    HierarchicalDatastore& operator=(const HierarchicalDatastore& o) {
        if (this == &o) return *this;
        dbl_store_t h = nullptr;
        check(dbl_store_clone(o.h_, &h));
        if (h_) dbl_store_destroy(h_);
        h_ = h;
        max_order = o.max_order;
        depth = o.depth;
        return *this;
    }

    NGramIndex prior{this, DBL_LAYER_PRIOR}, dynamic{this, DBL_LAYER_DYNAMIC}, rejected{this, DBL_LAYER_REJECTED};
    int max_order, depth;

    void set_rejected_enabled(bool on) { check(dbl_store_set_rejected_enabled(h_, on ? 1 : 0)); }
    // the device n-gram index over a layer's current sequences (build_prior builds the prior's); later
    // inserts into the layer are scanned until the next build — lookups are identical either way
    void build_index(int layer) { check(dbl_store_build_index(h_, layer)); }
    int64_t index_entries(int layer) const {
        int64_t v = 0;
        check(dbl_store_index_entries(h_, layer, &v));
        return v;
    }
    // device microseconds per lookup (back-to-back single-CTA lookups)
    double profile_lookup(std::span<const TokenId> context, int d, int iters = 100) {
        double us = 0;
        check(dbl_store_profile_lookup(h_, context.data(), static_cast<int>(context.size()), d, iters, &us));
        return us;
    }
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
    if (s_) {
        check(dbl_store_insert(s_->handle(), layer_, tokens.data(), static_cast<int>(tokens.size()), step));
        return;
    }
    if (tokens.empty()) throw std::invalid_argument("insert: empty token sequence");
    sequences.emplace_back(tokens.begin(), tokens.end());
    steps_.push_back(step);
}
inline size_t NGramIndex::occurrence_count() const {  // datastore.cpp:22-26
    if (s_) {
        int64_t ns = 0, nt = 0, occ = 0;
        check(dbl_store_layer_info(s_->handle(), layer_, &ns, &nt, &occ));
        return static_cast<size_t>(occ);
    }
    size_t total = 0;
    for (const TokenSeq& q : sequences)
        for (int k = 1; k <= max_order; ++k)
            if (static_cast<int>(q.size()) >= k) total += q.size() - k + 1;
    return total;
}
inline void NGramIndex::clear() {
    if (s_) {
        check(dbl_store_clear_layer(s_->handle(), layer_));
        return;
    }
    sequences.clear();
    steps_.clear();
}
inline std::vector<TokenSeq> NGramIndex::materialize() const {
    if (!s_) return sequences;
    int64_t ns = 0, nt = 0, occ = 0;
    check(dbl_store_layer_info(s_->handle(), layer_, &ns, &nt, &occ));
    std::vector<int32_t> toks(static_cast<size_t>(nt > 0 ? nt : 1)), lens(static_cast<size_t>(ns > 0 ? ns : 1));
    std::vector<int64_t> st(lens.size());
    check(dbl_store_layer_read(s_->handle(), layer_, toks.data(), static_cast<int64_t>(toks.size()), lens.data(),
                               st.data(), static_cast<int64_t>(lens.size())));
    std::vector<TokenSeq> out;
    size_t at = 0;
    for (int64_t i = 0; i < ns; ++i) {
        out.emplace_back(toks.begin() + static_cast<long>(at), toks.begin() + static_cast<long>(at + lens[i]));
        at += static_cast<size_t>(lens[i]);
    }
    return out;
}
inline std::vector<long> NGramIndex::steps() const {
    if (!s_) {
        if (steps_.size() == sequences.size()) return steps_;
        std::vector<long> v(sequences.size());
        for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<long>(i);
        return v;
    }
    int64_t ns = 0, nt = 0, occ = 0;
    check(dbl_store_layer_info(s_->handle(), layer_, &ns, &nt, &occ));
    std::vector<int32_t> toks(static_cast<size_t>(nt > 0 ? nt : 1)), lens(static_cast<size_t>(ns > 0 ? ns : 1));
    std::vector<int64_t> st(lens.size());
    check(dbl_store_layer_read(s_->handle(), layer_, toks.data(), static_cast<int64_t>(toks.size()), lens.data(),
                               st.data(), static_cast<int64_t>(lens.size())));
    return std::vector<long>(st.begin(), st.begin() + ns);
}
inline NGramIndex& NGramIndex::operator=(const NGramIndex& o) {
    if (this == &o) return *this;
    std::vector<TokenSeq> seqs = o.materialize();
    std::vector<long> st = o.steps();
    if (!s_) {
        max_order = o.max_order;
        sequences = std::move(seqs);
        steps_ = std::move(st);
        return *this;
    }
    bool dense = true;  // steps 0..n-1: one bulk upload (build_prior's shape)
    for (size_t i = 0; i < st.size(); ++i) dense = dense && st[i] == static_cast<long>(i);
    if (dense && layer_ == DBL_LAYER_PRIOR) {
        std::vector<int64_t> off{0};
        TokenSeq flat;
        for (const TokenSeq& q : seqs) {
            flat.insert(flat.end(), q.begin(), q.end());
            off.push_back(static_cast<int64_t>(flat.size()));
        }
        if (flat.empty()) flat.push_back(0);
        check(dbl_build_prior(s_->handle(), off.data(), flat.data(), static_cast<int>(seqs.size()), o.max_order,
                              static_cast<int>(seqs.size())));
    } else {
        check(dbl_store_clear_layer(s_->handle(), layer_));
        check(dbl_store_set_layer_order(s_->handle(), layer_, o.max_order));
        for (size_t i = 0; i < seqs.size(); ++i)
            check(dbl_store_insert(s_->handle(), layer_, seqs[i].data(), static_cast<int>(seqs[i].size()), st[i]));
    }
    max_order = o.max_order;
    return *this;
}

// build_prior (datastore.cpp:149-159): the first `rounds` corpus sequences, step = index, as an index
// value — `store.prior = build_prior(corpus, 3, 10)` loads it onto the device in one upload
inline NGramIndex build_prior(const std::vector<TokenSeq>& corpora, int max_order, int rounds) {
    if (rounds < 0) throw std::invalid_argument("build_prior: rounds must be >= 0");
    NGramIndex idx;
    idx.max_order = max_order;
    for (size_t i = 0; i < corpora.size() && static_cast<int>(i) < rounds; ++i) idx.insert(corpora[i], static_cast<long>(i));
    return idx;
}
// the same straight into store.prior
inline void build_prior(HierarchicalDatastore& store, const std::vector<TokenSeq>& corpora, int rounds) {
    store.prior = build_prior(corpora, store.max_order, rounds);
}

class Model {  // TableModel / transformer behind forward_batch (model.hpp:18-48)
  public:
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;
    Model(Model&& o) noexcept : forward_cost(o.forward_cost), h_(o.h_) { o.h_ = nullptr; }
    ~Model() { if (h_) dbl_model_destroy(h_); }
    int vocab_size() const {
        int v = 0;
        check(dbl_model_vocab(h_, &v));
        return v;
    }
    dbl_model_t handle() const { return h_; }
    double forward_cost = 1.0;  // TableModel::forward_cost (model.hpp:23): charged once per forward
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

struct SimClock {  // types.hpp:20-23
    double now = 0.0;
    void charge(double cost) { now += cost; }
};

struct LatencyConfig {  // pipeline.hpp:15-29
    double t_target = 1.0, t_draft = 0.25, t_lookup = 0.0, t_sync = 0.0;
    double speed_ratio() const {
        if (t_draft <= 0.0) throw std::invalid_argument("t_draft must be > 0");
        return t_target / t_draft;
    }
    void validate() const {
        if (t_target < 0.0 || t_draft <= 0.0 || t_lookup < 0.0 || t_sync < 0.0)
            throw std::invalid_argument("latency values out of range");
    }
};

enum class Mode { PreVerify, PostVerify };  // pipeline.hpp:31
enum class Engine { Serial, Concurrent };   // pipeline.hpp:32 (the device always overlaps; results identical)
inline const char* to_string(Mode m) { return m == Mode::PreVerify ? "pre_verify" : "post_verify"; }

struct PipelineOptions {  // pipeline.hpp:36-44
    int gamma = 4, depth = 10;
    bool draft_retrieval = true, target_retrieval = true;
    Engine engine = Engine::Serial;
    SamplerConfig sampler{};
    LatencyConfig latency{};
};

using RunMetrics = dbl_run_metrics;  // RunMetrics (pipeline.hpp:73-82) + device timing fields

struct RoundTrace {  // pipeline.hpp:57-71
    long round = 0;
    std::string mode;
    int pending = 0, draft_len = 0;
    std::vector<int> draft_matched;
    int target_matched = -1;
    std::string target_source;
    int accepted_pending = 0;
    bool pending_reject = false, rejected = false;
    int committed_count = 0;
    std::string kind;
    double clock_delta = 0.0;
};

struct RunResult {  // pipeline.hpp:84-88
    TokenSeq output;
    RunMetrics metrics{};
    std::vector<RoundTrace> traces;
    std::string jsonl;  // traces_to_jsonl(traces)
};

namespace detail {
inline dbl_pipeline_options c_options(const PipelineOptions& o) {
    return dbl_pipeline_options{o.gamma, o.depth, o.draft_retrieval, o.target_retrieval,
                                o.engine == Engine::Concurrent, o.latency.t_target, o.latency.t_draft,
                                o.latency.t_lookup, o.latency.t_sync, 1, o.sampler.temperature,
                                o.sampler.rng_seed};
}
inline const char* const kModes[] = {"pre_verify", "post_verify", "ar", "serial"};
inline const char* const kKinds[] = {"pending_reject", "extend_keep_draft", "extend_draft_subsumed",
                                     "extend_drop_draft", "ar_step", "reject", "all_accepted"};
inline const char* const kSources[] = {"prior", "dynamic", "rejected", "context", "miss"};
inline int index_of(const char* const* names, int n, const std::string& v) {
    for (int i = 0; i < n; ++i)
        if (v == names[i]) return i;
    throw std::invalid_argument("unknown trace label '" + v + "'");
}
inline RoundTrace from_c(const dbl_round_trace& c) {
    RoundTrace t;
    t.round = static_cast<long>(c.round);
    t.mode = kModes[c.mode];
    t.pending = c.pending;
    t.draft_len = c.draft_len;
    t.draft_matched.assign(c.draft_matched, c.draft_matched + c.n_draft_matched);
    t.target_matched = c.target_matched;
    t.target_source = kSources[c.target_source];
    t.accepted_pending = c.accepted_pending;
    t.pending_reject = c.pending_reject != 0;
    t.rejected = c.rejected != 0;
    t.committed_count = c.committed_count;
    t.kind = kKinds[c.kind];
    t.clock_delta = c.clock_delta;
    return t;
}
inline dbl_round_trace to_c(const RoundTrace& t) {
    dbl_round_trace c{};
    c.round = t.round;
    c.mode = index_of(kModes, 4, t.mode.empty() ? "pre_verify" : t.mode);
    c.pending = t.pending;
    c.draft_len = t.draft_len;
    if (t.draft_matched.size() > DBL_MAX_SEGS) throw std::invalid_argument("more than DBL_MAX_SEGS segments");
    c.n_draft_matched = static_cast<int>(t.draft_matched.size());
    for (size_t k = 0; k < t.draft_matched.size(); ++k) c.draft_matched[k] = t.draft_matched[k];
    c.target_matched = t.target_matched;
    c.target_source = index_of(kSources, 5, t.target_source.empty() ? "miss" : t.target_source);
    c.accepted_pending = t.accepted_pending;
    c.pending_reject = t.pending_reject;
    c.rejected = t.rejected;
    c.committed_count = t.committed_count;
    c.kind = index_of(kKinds, 7, t.kind.empty() ? "extend_draft_subsumed" : t.kind);
    c.clock_delta = t.clock_delta;
    return c;
}
inline std::vector<dbl_round_trace> to_c(const std::vector<RoundTrace>& ts) {
    std::vector<dbl_round_trace> v;
    for (const RoundTrace& t : ts) v.push_back(to_c(t));
    if (v.empty()) v.push_back(dbl_round_trace{});
    return v;
}
// RunResult::traces of this thread's last run (dbl_last_run_traces)
inline std::vector<RoundTrace> last_traces() {
    int64_t n = 0;
    check(dbl_last_run_traces(nullptr, 0, &n));
    std::vector<dbl_round_trace> c(static_cast<size_t>(n > 0 ? n : 1));
    check(dbl_last_run_traces(c.data(), static_cast<int64_t>(c.size()), &n));
    std::vector<RoundTrace> out;
    for (int64_t i = 0; i < n; ++i) out.push_back(from_c(c[i]));
    return out;
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
    r.traces = detail::last_traces();
    r.jsonl.resize(static_cast<size_t>(jl) + 1);
    check(dbl_last_run_jsonl(r.jsonl.data(), static_cast<int64_t>(r.jsonl.size()), &jl));
    r.jsonl.resize(static_cast<size_t>(jl));
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

// sampled decoding at wide vocabularies on the reference-exact path (dbl_set_exact_sampling)
inline void set_exact_sampling(bool on = true) { check(dbl_set_exact_sampling(on ? 1 : 0)); }

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
    r.traces = detail::last_traces();
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

// ------------------------------------------------------------------ model-level (model.hpp:29-48)
// forward (model.cpp:30-35): the next-token distribution after ctx; charges forward_cost once
inline ProbVector forward(const Model& m, std::span<const TokenId> ctx, SimClock* clock = nullptr) {
    ProbVector p(static_cast<size_t>(m.vocab_size()));
    check(dbl_forward_dists(m.handle(), ctx.data(), static_cast<int>(ctx.size()), nullptr, 0, p.data()));
    if (clock) clock->charge(m.forward_cost);
    return p;
}
// forward_batch with the reference's clock argument: |cands|+1 rows, forward_cost charged once
inline std::vector<ProbVector> forward_batch(const Model& m, std::span<const TokenId> ctx,
                                             std::span<const TokenId> cands, SimClock* clock) {
    std::vector<ProbVector> rows = forward_batch(m, ctx, cands);
    if (clock) clock->charge(m.forward_cost);
    return rows;
}
inline ProbVector tempered(const ProbVector& dist, double temperature) {  // model.cpp:55-68
    ProbVector out(dist.size());
    check(dbl_tempered(dist.data(), static_cast<int>(dist.size()), temperature, 0, out.data()));
    return out;
}
inline TokenId argmax_token(const ProbVector& dist) {  // model.cpp:70-81
    TokenId t = 0;
    check(dbl_argmax_token(dist.data(), static_cast<int>(dist.size()), 0, &t));
    return t;
}
inline TokenId sample(const ProbVector& dist, const SamplerConfig& cfg, Rng& rng) {  // model.cpp:83-97
    TokenId t = 0;
    check(dbl_sample(dist.data(), static_cast<int>(dist.size()), cfg.temperature, rng.handle(), 0, &t));
    return t;
}

// ------------------------------------------------------------------ drafter (speculation.hpp:12-59)
struct RetrievalResult {
    TokenSeq emitted;  // matched prefix + correction, length matched_len + 1
    int matched_len = 0;
    std::vector<ProbVector> probs;
    LookupSource source = LookupSource::Miss;
};
struct DraftChain {
    std::vector<RetrievalResult> segments;
    TokenSeq tokens;
    std::vector<ProbVector> probs;
    int total_len = 0;
};

inline RetrievalResult accept_with_model(std::span<const ProbVector> dists, std::span<const TokenId> cands,
                                         const SamplerConfig& cfg, Rng& rng) {  // speculation.cpp:7-52
    const detail::Rows d(dists);
    TokenSeq em(cands.size() + 1);
    std::vector<double> pr(d.data.size());
    dbl_retrieval_result res{};
    check(dbl_accept_with_model(d.data.data(), d.off.data(), d.n(), cands.data(), static_cast<int>(cands.size()),
                                cfg.temperature, rng.handle(), 0, em.data(), static_cast<int>(em.size()), pr.data(),
                                static_cast<int64_t>(pr.size()), &res));
    RetrievalResult r;
    r.emitted.assign(em.begin(), em.begin() + res.n_emitted);
    r.matched_len = res.matched_len;
    for (int i = 0; i < res.n_probs; ++i)
        r.probs.emplace_back(pr.begin() + d.off[i], pr.begin() + d.off[i + 1]);
    return r;
}

inline RetrievalResult retrieval_forward(const Model& model, const HierarchicalDatastore& store,
                                         std::span<const TokenId> context, int depth, const SamplerConfig& cfg,
                                         Rng& rng, SimClock* clock = nullptr,
                                         bool use_retrieval = true) {  // speculation.cpp:54-66
    const size_t V = static_cast<size_t>(model.vocab_size());
    TokenSeq em(static_cast<size_t>(depth > 0 ? depth : 0) + 1);
    std::vector<double> pr(em.size() * V);
    dbl_retrieval_result res{};
    check(dbl_retrieval_forward(model.handle(), store.handle(), context.data(), static_cast<int>(context.size()), depth,
                                cfg.temperature, rng.handle(), use_retrieval, em.data(), static_cast<int>(em.size()),
                                pr.data(), static_cast<int64_t>(pr.size()), &res));
    if (clock) clock->charge(model.forward_cost);
    RetrievalResult r;
    r.emitted.assign(em.begin(), em.begin() + res.n_emitted);
    r.matched_len = res.matched_len;
    r.source = static_cast<LookupSource>(res.source);
    for (int i = 0; i < res.n_probs; ++i)
        r.probs.emplace_back(pr.begin() + static_cast<long>(i * V), pr.begin() + static_cast<long>((i + 1) * V));
    return r;
}

inline DraftChain iterative_draft(const Model& model, const HierarchicalDatastore& store,
                                  std::span<const TokenId> context, int gamma, int depth, const SamplerConfig& cfg,
                                  Rng& rng, SimClock* clock = nullptr,
                                  bool use_retrieval = true) {  // speculation.cpp:68-86
    if (gamma < 1) throw std::invalid_argument("iterative_draft: gamma must be >= 1");
    const size_t V = static_cast<size_t>(model.vocab_size());
    const size_t cap = static_cast<size_t>(gamma) * (static_cast<size_t>(depth > 0 ? depth : 0) + 1);
    TokenSeq toks(cap);
    std::vector<double> pr(cap * V);
    std::vector<dbl_retrieval_result> segs(static_cast<size_t>(gamma));
    int n = 0;
    check(dbl_iterative_draft(model.handle(), store.handle(), context.data(), static_cast<int>(context.size()), gamma,
                              depth, cfg.temperature, rng.handle(), use_retrieval, segs.data(), toks.data(),
                              static_cast<int>(toks.size()), &n, pr.data(), static_cast<int64_t>(pr.size())));
    DraftChain ch;
    ch.tokens.assign(toks.begin(), toks.begin() + n);
    for (int i = 0; i < n; ++i)
        ch.probs.emplace_back(pr.begin() + static_cast<long>(i * V), pr.begin() + static_cast<long>((i + 1) * V));
    size_t at = 0;
    for (const dbl_retrieval_result& g : segs) {
        RetrievalResult r;
        r.emitted.assign(ch.tokens.begin() + static_cast<long>(at), ch.tokens.begin() + static_cast<long>(at + g.n_emitted));
        r.probs.assign(ch.probs.begin() + static_cast<long>(at), ch.probs.begin() + static_cast<long>(at + g.n_emitted));
        r.matched_len = g.matched_len;
        r.source = static_cast<LookupSource>(g.source);
        at += static_cast<size_t>(g.n_emitted);
        ch.segments.push_back(std::move(r));
        if (clock) clock->charge(model.forward_cost);
    }
    ch.total_len = n;
    return ch;
}

inline double measure_amt(std::span<const RetrievalResult> traces) {  // speculation.cpp:88-94
    std::vector<int32_t> m;
    for (const RetrievalResult& r : traces) m.push_back(r.matched_len);
    double out = 0.0;
    check(dbl_measure_amt(m.data(), static_cast<int>(m.size()), &out));
    return out;
}

// ------------------------------------------------------------------ decoder state machine (pipeline.hpp)
// A run_round session: the device lanes (token buffers + KV) a PipelineState runs on between rounds.
class Session {
  public:
    Session(const Model& draft, const Model& target) : draft_(draft.handle()), target_(target.handle()) {
        check(dbl_session_create(draft_, target_, &h_));
    }
    ~Session() { dbl_session_destroy(h_); }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    dbl_session_t handle() const { return h_; }
    bool serves(const Model& d, const Model& t) const { return d.handle() == draft_ && t.handle() == target_; }

  private:
    dbl_model_t draft_, target_;
    dbl_session_t h_ = nullptr;
};

struct PipelineState {  // pipeline.hpp:46-55
    TokenSeq committed;
    TokenSeq speculative;
    std::vector<ProbVector> spec_probs;  // T > 0: the rows; greedy: |speculative| rows (never read)
    Mode mode = Mode::PreVerify;
    int prev_tokens = 0;
    long round = 0;
    SimClock clock;
    long last_committed_len = 0;
    std::shared_ptr<Session> session;    // the lanes this state last ran on (shared by copies; any state
                                         // re-synchronises them by longest common prefix)
};

inline void rollback(PipelineState& state, long keep_len) {  // pipeline.cpp:15-30
    dbl_pipeline_state c{};
    c.committed = state.committed.data();
    c.n_committed = c.committed_cap = static_cast<int64_t>(state.committed.size());
    c.n_speculative = c.speculative_cap = static_cast<int64_t>(state.speculative.size());
    c.n_spec_probs = static_cast<int64_t>(state.spec_probs.size());
    c.mode = state.mode == Mode::PostVerify;
    c.last_committed_len = state.last_committed_len;
    check(dbl_rollback(&c, keep_len));
    state.committed.resize(static_cast<size_t>(c.n_committed));
    state.speculative.clear();
    state.spec_probs.clear();
    state.mode = Mode::PreVerify;
}

inline RoundTrace run_round(PipelineState& state, const Model& draft_model, const Model& target_model,
                            HierarchicalDatastore& store, const PipelineOptions& opts) {  // pipeline.cpp:223-262
    if (!state.session || !state.session->serves(draft_model, target_model))
        state.session = std::make_shared<Session>(draft_model, target_model);
    const int64_t gd = static_cast<int64_t>(opts.gamma) * (opts.depth + 1);
    const size_t V = static_cast<size_t>(target_model.vocab_size());
    TokenSeq com = state.committed, spec = state.speculative;
    com.resize(state.committed.size() + state.speculative.size() + static_cast<size_t>(opts.depth > 0 ? opts.depth : 0) + 1);
    spec.resize(static_cast<size_t>(std::max<int64_t>(gd, static_cast<int64_t>(state.speculative.size()))) + 1);
    dbl_pipeline_state c{};
    c.committed = com.data();
    c.n_committed = static_cast<int64_t>(state.committed.size());
    c.committed_cap = static_cast<int64_t>(com.size());
    c.speculative = spec.data();
    c.n_speculative = static_cast<int64_t>(state.speculative.size());
    c.speculative_cap = static_cast<int64_t>(spec.size());
    c.n_spec_probs = static_cast<int64_t>(state.spec_probs.size());
    std::vector<double> rows;
    const bool sampled = opts.sampler.temperature != 0.0;
    if (sampled) {
        const size_t cap_rows = std::max<size_t>(static_cast<size_t>(gd), state.speculative.size()) + 1;
        rows.assign(cap_rows * V, 0.0);
        bool full = state.spec_probs.size() == state.speculative.size();
        for (size_t i = 0; full && i < state.spec_probs.size(); ++i) {
            if (state.spec_probs[i].size() != V) throw std::invalid_argument("spec_probs row size != vocab");
            std::memcpy(rows.data() + i * V, state.spec_probs[i].data(), V * sizeof(double));
        }
        c.spec_probs = rows.data();
        c.spec_probs_cap = static_cast<int64_t>(cap_rows);
    }
    c.mode = state.mode == Mode::PostVerify;
    c.prev_tokens = state.prev_tokens;
    c.round = state.round;
    c.clock = state.clock.now;
    c.last_committed_len = state.last_committed_len;
    const dbl_pipeline_options o = detail::c_options(opts);
    dbl_round_trace tr{};
    check(dbl_run_round(state.session->handle(), store.handle(), &o, &c, &tr));
    state.committed.assign(com.begin(), com.begin() + c.n_committed);
    state.speculative.assign(spec.begin(), spec.begin() + c.n_speculative);
    state.spec_probs.assign(static_cast<size_t>(c.n_spec_probs), ProbVector{});
    if (sampled)
        for (int64_t i = 0; i < c.n_spec_probs; ++i)
            state.spec_probs[i].assign(rows.begin() + static_cast<long>(i * V), rows.begin() + static_cast<long>((i + 1) * V));
    state.mode = c.mode ? Mode::PostVerify : Mode::PreVerify;
    state.prev_tokens = c.prev_tokens;
    state.round = static_cast<long>(c.round);
    state.clock.now = c.clock;
    state.last_committed_len = static_cast<long>(c.last_committed_len);
    return detail::from_c(tr);
}

inline RunMetrics compute_metrics(const std::vector<RoundTrace>& traces, const LatencyConfig& latency) {
    const std::vector<dbl_round_trace> c = detail::to_c(traces);  // pipeline.cpp:325-371
    RunMetrics m{};
    check(dbl_compute_metrics(c.data(), static_cast<int>(traces.size()), latency.t_target, &m));
    return m;
}
inline std::string traces_to_jsonl(const std::vector<RoundTrace>& traces) {  // pipeline.cpp:373-394
    const std::vector<dbl_round_trace> c = detail::to_c(traces);
    int64_t n = 0;
    check(dbl_traces_to_jsonl(c.data(), static_cast<int>(traces.size()), nullptr, 0, &n));
    std::string s(static_cast<size_t>(n) + 1, '\0');
    check(dbl_traces_to_jsonl(c.data(), static_cast<int>(traces.size()), s.data(), static_cast<int64_t>(s.size()), &n));
    s.resize(static_cast<size_t>(n));
    return s;
}
inline void write_traces(const std::vector<RoundTrace>& traces, const std::string& path) {  // pipeline.cpp:396-400
    const std::vector<dbl_round_trace> c = detail::to_c(traces);
    check(dbl_write_traces(c.data(), static_cast<int>(traces.size()), path.c_str()));
}

}  // namespace specpar_b200
