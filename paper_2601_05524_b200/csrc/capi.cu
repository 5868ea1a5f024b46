// The extern "C" boundary (include/double_b200.h): status codes + thread-local last error; the
// C++ exceptions of the engine never cross it.
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>

#include "decoder.cuh"
#include "store.cuh"
#include "table_model.cuh"
#include "transformer.cuh"
#include "tp.cuh"
#include "fwd.cuh"
#include "verify.cuh"
#include "gemm.cuh"
#include "sampling.cuh"
#include "lane.cuh"
#include "tf_kernels.cuh"
#include <cuda_bf16.h>

struct dbl_store_s {
    std::unique_ptr<dbl::DeviceStore> impl;
};
struct dbl_model_s {
    std::unique_ptr<dbl::Model> impl;
};
struct dbl_rng_s {
    std::unique_ptr<dbl::DeviceRng> impl;
};

namespace {
thread_local std::string g_last_error;
thread_local std::vector<int32_t> g_last_log;
thread_local std::string g_last_jsonl;  // traces_to_jsonl of this thread's last single-sequence run
thread_local std::vector<dbl::Trace> g_last_traces;  // RunResult::traces of that run

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return DBL_OK;
    } catch (const dbl::Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("out of memory: ") + e.what();
        return DBL_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DBL_RUNTIME_ERROR;
    }
}

void need(const void* p, const char* what) {
    if (!p) dbl::throw_invalid(std::string("null ") + what);
}

int copy_run(const dbl::RunOutput& r, int32_t* out, int cap, int* n_out, dbl_run_metrics* metrics,
             char* jsonl, int64_t jsonl_cap, int64_t* jsonl_len) {
    if (static_cast<int>(r.output.size()) > cap) dbl::throw_invalid("output buffer too small");
    if (out && !r.output.empty()) std::memcpy(out, r.output.data(), r.output.size() * 4);
    if (n_out) *n_out = static_cast<int>(r.output.size());
    if (metrics) *metrics = r.metrics;
    g_last_traces = r.traces;
    if (jsonl || jsonl_len) {
        // tokens and metrics are already out; the text stays readable through dbl_last_run_jsonl, so a
        // short buffer costs a second copy, never the (already mutated-store) run
        g_last_jsonl = dbl::traces_to_jsonl(r.traces);
        const std::string& js = g_last_jsonl;
        if (jsonl_len) *jsonl_len = static_cast<int64_t>(js.size());
        if (jsonl) {
            if (static_cast<int64_t>(js.size()) + 1 > jsonl_cap)
                dbl::throw_invalid("jsonl buffer too small (need " + std::to_string(js.size() + 1) +
                                   " bytes; tokens and metrics were written, the text is in dbl_last_run_jsonl)");
            std::memcpy(jsonl, js.c_str(), js.size() + 1);
        }
    }
    return 0;
}
}  // namespace

namespace dbl {
long long& launch_counter() {
    thread_local long long n = 0;
    return n;
}
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DBL_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
void require_device(int device) {
    static std::mutex mu;
    static std::vector<int> ok;  // per device: 0 unknown, 1 sm_100, 2 other
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        throw Error(DBL_CUDA_ERROR, "no CUDA device visible (libdouble_b200 has no CPU fallback)");
    }
    if (device < 0 || device >= n) throw Error(DBL_INVALID_ARGUMENT, "device index out of range");
    std::lock_guard<std::mutex> lk(mu);
    if (static_cast<int>(ok.size()) < n) ok.resize(n, 0);
    if (!ok[device]) {
        int major = 0;
        CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        ok[device] = major == 10 ? 1 : 2;
    }
    if (ok[device] != 1) throw Error(DBL_CUDA_ERROR, "libdouble_b200 is built for sm_100a (B200) only");
}

namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;  // size class -> cached mapped pinned blocks
size_t g_pin_cached = 0;
constexpr size_t kPinCacheMax = size_t(512) << 20;
}  // namespace

void* pinned_get(size_t bytes, size_t* got) {
    size_t cls = 4096;
    while (cls < bytes) cls <<= 1;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.find(cls);
        if (it != g_pin_free.end()) {
            void* p = it->second;
            g_pin_free.erase(it);
            g_pin_cached -= cls;
            *got = cls;
            return p;
        }
    }
    void* p = nullptr;
    CUDA_CHECK(cudaHostAlloc(&p, cls, cudaHostAllocMapped | cudaHostAllocPortable));
    *got = cls;
    return p;
}

void pinned_put(void* p, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        if (g_pin_cached + bytes <= kPinCacheMax) {
            g_pin_free.emplace(bytes, p);
            g_pin_cached += bytes;
            return;
        }
    }
    cudaFreeHost(p);
}
}  // namespace dbl

extern "C" {

const char* dbl_last_error(void) { return g_last_error.c_str(); }
int dbl_version(void) { return 1; }
int dbl_device_ok(void) {
    try {
        dbl::require_device(0);
        return 1;
    } catch (...) {
        return 0;
    }
}

// ------------------------------------------------------------------------------- datastore
int dbl_store_create(int max_order, int depth, int device, dbl_store_t* out) {
    return guarded([&] {
        need(out, "out");
        auto* s = new dbl_store_s;
        try {
            s->impl = std::make_unique<dbl::DeviceStore>(max_order, depth, device);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}
int dbl_store_destroy(dbl_store_t s) {
    return guarded([&] { delete s; });
}
int dbl_store_set_rejected_enabled(dbl_store_t s, int enabled) {
    return guarded([&] { need(s, "store"); s->impl->set_rejected_enabled(enabled != 0, 0); });
}
int dbl_store_set_layer_order(dbl_store_t s, int layer, int max_order) {
    return guarded([&] { need(s, "store"); s->impl->set_layer_order(layer, max_order, 0); });
}
int dbl_store_insert(dbl_store_t s, int layer, const int32_t* tokens, int n, int64_t step) {
    return guarded([&] {
        need(s, "store");
        if (n > 0) need(tokens, "tokens");
        s->impl->insert(layer, tokens, n, step, 0);
    });
}
int dbl_store_record(dbl_store_t s, int layer, const int32_t* tokens, int n) {
    return guarded([&] {
        need(s, "store");
        if (layer != DBL_LAYER_DYNAMIC && layer != DBL_LAYER_REJECTED)
            dbl::throw_invalid("record: layer must be dynamic or rejected");
        if (n > 0) need(tokens, "tokens");
        s->impl->record(layer, tokens, n, 0);
    });
}
int dbl_store_flush_session(dbl_store_t s) {
    return guarded([&] { need(s, "store"); s->impl->flush_session(0); });
}
int dbl_store_clear_layer(dbl_store_t s, int layer) {
    return guarded([&] { need(s, "store"); s->impl->clear_layer(layer, 0); });
}
int dbl_store_build_index(dbl_store_t s, int layer) {
    return guarded([&] { need(s, "store"); s->impl->build_index(layer, 0); });
}
int dbl_store_index_entries(dbl_store_t s, int layer, int64_t* entries) {
    return guarded([&] { need(s, "store"); need(entries, "entries"); *entries = s->impl->index_entries(layer); });
}
int dbl_store_profile_lookup(dbl_store_t s, const int32_t* ctx, int L, int d, int iters, double* us) {
    return guarded([&] {
        need(s, "store");
        need(ctx, "ctx");
        need(us, "us_per_lookup");
        if (L <= 0) dbl::throw_invalid("lookup: empty context");
        if (iters < 1) dbl::throw_invalid("iters must be >= 1");
        *us = s->impl->profile_lookup(ctx, L, d, iters);
    });
}
int dbl_store_get_step(dbl_store_t s, int64_t* step) {
    return guarded([&] { need(s, "store"); need(step, "step"); *step = s->impl->step(); });
}
int dbl_store_set_step(dbl_store_t s, int64_t step) {
    return guarded([&] { need(s, "store"); s->impl->set_step(step); });
}
int dbl_store_layer_info(dbl_store_t s, int layer, int64_t* n_seqs, int64_t* n_tokens, int64_t* occ) {
    return guarded([&] { need(s, "store"); s->impl->layer_info(layer, n_seqs, n_tokens, occ); });
}
int dbl_store_layer_read(dbl_store_t s, int layer, int32_t* tokens, int64_t tok_cap, int32_t* seq_lens,
                         int64_t* steps, int64_t seq_cap) {
    return guarded([&] {
        need(s, "store");
        s->impl->layer_read(layer, tokens, tok_cap, seq_lens, steps, seq_cap, 0);
    });
}
int dbl_store_lookup(dbl_store_t s, const int32_t* ctx, int L, int d, int32_t* cands, int cap,
                     int* n_cands, int* source, int* matched_order) {
    return guarded([&] {
        need(s, "store");
        if (L <= 0) dbl::throw_invalid("lookup: empty context");
        need(ctx, "ctx");
        const int dcap = std::max(d, 1);
        std::vector<int32_t> c(dcap);
        const int64_t off[2] = {0, L};
        int32_t n = 0, src = 0, ord = 0;
        s->impl->lookup_batch(1, off, ctx, &d, dcap, c.data(), &n, &src, &ord, 0);
        if (n > cap) dbl::throw_invalid("candidate buffer too small");
        if (n) std::memcpy(cands, c.data(), n * 4);
        if (n_cands) *n_cands = n;
        if (source) *source = src;
        if (matched_order) *matched_order = ord;
    });
}
int dbl_store_lookup_batch(dbl_store_t s, int n_q, const int64_t* q_offsets, const int32_t* q_tokens,
                           const int32_t* depths, int d_cap, int32_t* out_cands, int32_t* out_n,
                           int32_t* out_source, int32_t* out_order) {
    return guarded([&] {
        need(s, "store");
        s->impl->lookup_batch(n_q, q_offsets, q_tokens, depths, d_cap, out_cands, out_n, out_source,
                              out_order, 0);
    });
}
int dbl_store_stats(dbl_store_t s, int64_t out[6]) {
    return guarded([&] { need(s, "store"); s->impl->stats(out, 0); });
}

// ---------------------------------------------------------------------------------- models
int dbl_table_create(int order, int vocab, int64_t n_rows, const int32_t* windows, const double* probs,
                     const double* fallback, int device, dbl_model_t* out) {
    return guarded([&] {
        need(out, "out");
        need(fallback, "fallback");
        if (n_rows > 0) { need(windows, "windows"); need(probs, "probs"); }
        auto m = std::make_unique<dbl_model_s>();
        m->impl = std::make_unique<dbl::TableModel>(order, vocab, n_rows, windows, probs, fallback, device);
        *out = m.release();
    });
}
int dbl_transformer_create(const dbl_transformer_config* cfg, int device, void* nccl_comm, dbl_model_t* out) {
    return guarded([&] {
        need(cfg, "config");
        need(out, "out");
        auto m = std::make_unique<dbl_model_s>();
        m->impl = std::make_unique<dbl::Transformer>(*cfg, device, nccl_comm);
        *out = m.release();
    });
}
int dbl_tp_ipc_export(dbl_model_t shard, void* out, int64_t cap) {
    return guarded([&] {
        need(shard, "shard");
        need(out, "out");
        if (cap < static_cast<int64_t>(4 * sizeof(cudaIpcMemHandle_t))) dbl::throw_invalid("handle buffer too small");
        auto* t = dynamic_cast<dbl::Transformer*>(shard->impl.get());
        if (!t) dbl::throw_invalid("not a transformer shard");
        t->ipc_export(out);
    });
}
int dbl_tp_ipc_import(dbl_model_t shard, const void* all, int world) {
    return guarded([&] {
        need(shard, "shard");
        need(all, "handles");
        auto* t = dynamic_cast<dbl::Transformer*>(shard->impl.get());
        if (!t) dbl::throw_invalid("not a transformer shard");
        t->ipc_import(all, world);
    });
}
int dbl_tp_transformer_create(const dbl_transformer_config* cfg, const int* devices, int world, dbl_model_t* out) {
    return guarded([&] {
        need(cfg, "config");
        need(devices, "devices");
        need(out, "out");
        if (world < 2 || world > dbl::kMaxTpRanks) dbl::throw_invalid("tensor parallel: 2..8 shards");
        auto m = std::make_unique<dbl_model_s>();
        m->impl = std::make_unique<dbl::TpTransformer>(*cfg, std::vector<int>(devices, devices + world));
        *out = m.release();
    });
}
int dbl_model_destroy(dbl_model_t m) {
    return guarded([&] { delete m; });
}
int dbl_model_vocab(dbl_model_t m, int* vocab) {
    return guarded([&] { need(m, "model"); need(vocab, "vocab"); *vocab = m->impl->vocab(); });
}
int dbl_model_weight_bytes(dbl_model_t m, int64_t* bytes) {
    return guarded([&] { need(m, "model"); need(bytes, "bytes"); *bytes = m->impl->weight_bytes(); });
}
int dbl_forward_argmax(dbl_model_t m, const int32_t* ctx, int L, const int32_t* cands, int c, int32_t* out) {
    return guarded([&] {
        need(m, "model");
        need(out, "out");
        dbl::forward_stateless(*m->impl, ctx, L, cands, c, out, nullptr);
    });
}
int dbl_forward_logits(dbl_model_t m, const int32_t* ctx, int L, const int32_t* cands, int c, float* out) {
    return guarded([&] {
        need(m, "model");
        need(out, "out");
        std::vector<int32_t> am(c + 1);
        dbl::forward_stateless(*m->impl, ctx, L, cands, c, am.data(), out);
    });
}
int dbl_forward_dists(dbl_model_t m, const int32_t* ctx, int L, const int32_t* cands, int c, double* out) {
    return guarded([&] {
        need(m, "model");
        need(out, "out");
        std::vector<int32_t> am(c + 1);
        dbl::forward_stateless(*m->impl, ctx, L, cands, c, am.data(), nullptr, out);
    });
}
int dbl_transformer_get_weight(dbl_model_t m, const char* name, int layer, uint16_t* out, int64_t numel) {
    return guarded([&] {
        need(m, "model");
        need(name, "name");
        auto* t = dynamic_cast<dbl::Transformer*>(m->impl.get());
        if (!t) dbl::throw_invalid("not a transformer model");
        t->get_weight(name, layer, out, numel);
    });
}

// ------------------------------------------------------------------------ model-level helpers
int dbl_tempered(const double* dist, int n, double temperature, int device, double* out) {
    return guarded([&] { dbl::tempered(dist, n, temperature, out, device); });
}
int dbl_argmax_token(const double* dist, int n, int device, int32_t* out) {
    return guarded([&] {
        need(out, "out");
        if (n <= 0) dbl::throw_runtime("degenerate distribution");  // model.cpp:79 (empty row)
        need(dist, "dist");
        const int64_t off[2] = {0, n};
        dbl::argmax_rows(dist, off, 1, out, device);
    });
}
int dbl_argmax_rows(const double* probs, const int64_t* off, int n_rows, int device, int32_t* out) {
    return guarded([&] {
        if (n_rows < 0) dbl::throw_invalid("negative row count");
        if (n_rows == 0) return;
        need(off, "offsets");
        need(out, "out");
        for (int r = 0; r < n_rows; ++r)
            if (off[r + 1] <= off[r]) dbl::throw_runtime("degenerate distribution");
        dbl::argmax_rows(probs, off, n_rows, out, device);
    });
}
int dbl_sample(const double* dist, int n, double temperature, dbl_rng_t r, int device, int32_t* out) {
    return guarded([&] {
        need(out, "out");
        *out = dbl::sample(dist, n, temperature, r ? r->impl.get() : nullptr, r ? r->impl->device() : device);
    });
}

// ------------------------------------------------------------------------------------ drafter
namespace {
void copy_retrieval(const std::vector<int32_t>& emitted, int matched, int source, int n_probs,
                    const std::vector<double>& probs, int32_t* out, int cap, double* pout, int64_t pcap,
                    dbl_retrieval_result* res) {
    if (static_cast<int>(emitted.size()) > cap) dbl::throw_invalid("emitted buffer too small");
    if (!emitted.empty()) std::memcpy(out, emitted.data(), emitted.size() * 4);
    if (pout) {
        if (static_cast<int64_t>(probs.size()) > pcap) dbl::throw_invalid("probs buffer too small");
        if (!probs.empty()) std::memcpy(pout, probs.data(), probs.size() * sizeof(double));
    }
    if (res) *res = dbl_retrieval_result{matched, static_cast<int>(emitted.size()), source, n_probs};
}
}  // namespace

int dbl_accept_with_model(const double* dists, const int64_t* dist_off, int n_dists, const int32_t* cands, int c,
                          double temperature, dbl_rng_t r, int device, int32_t* emitted, int emitted_cap,
                          double* probs, int64_t probs_cap, dbl_retrieval_result* res) {
    return guarded([&] {
        need(emitted, "emitted");
        if (n_dists > 0) {
            need(dists, "dists");
            need(dist_off, "dist offsets");
        }
        const dbl::AcceptOut a = dbl::accept_with_model(dists, dist_off, n_dists, cands, c, temperature,
                                                        r ? r->impl.get() : nullptr, device, probs != nullptr);
        copy_retrieval(a.emitted, a.matched_len, DBL_SRC_MISS, a.n_probs, a.probs, emitted, emitted_cap, probs,
                       probs_cap, res);
    });
}
int dbl_retrieval_forward(dbl_model_t m, dbl_store_t st, const int32_t* ctx, int L, int depth, double temperature,
                          dbl_rng_t r, int use_retrieval, int32_t* emitted, int emitted_cap, double* probs,
                          int64_t probs_cap, dbl_retrieval_result* res) {
    return guarded([&] {
        need(m, "model");
        need(emitted, "emitted");
        if (L > 0) need(ctx, "ctx");
        if (use_retrieval) need(st, "store");
        const dbl::RetrievalOut o =
            dbl::retrieval_forward(*m->impl, st ? st->impl.get() : nullptr, ctx, L, depth, temperature,
                                   r ? r->impl.get() : nullptr, use_retrieval != 0, probs != nullptr);
        copy_retrieval(o.emitted, o.matched_len, o.source, o.n_probs, o.probs, emitted, emitted_cap, probs, probs_cap,
                       res);
    });
}
int dbl_iterative_draft(dbl_model_t m, dbl_store_t st, const int32_t* ctx, int L, int gamma, int depth,
                        double temperature, dbl_rng_t r, int use_retrieval, dbl_retrieval_result* segs,
                        int32_t* tokens, int tokens_cap, int* n_tokens, double* probs, int64_t probs_cap) {
    return guarded([&] {  // speculation.cpp:68-86
        need(m, "model");
        if (gamma < 1) dbl::throw_invalid("iterative_draft: gamma must be >= 1");
        need(tokens, "tokens");
        if (L > 0) need(ctx, "ctx");
        if (use_retrieval) need(st, "store");
        std::vector<int32_t> grown(ctx, ctx + std::max(L, 0)), flat;
        std::vector<double> rows;
        std::vector<dbl_retrieval_result> rs;
        for (int j = 0; j < gamma; ++j) {
            const dbl::RetrievalOut o = dbl::retrieval_forward(
                *m->impl, st ? st->impl.get() : nullptr, grown.data(), static_cast<int>(grown.size()), depth,
                temperature, r ? r->impl.get() : nullptr, use_retrieval != 0, probs != nullptr);
            grown.insert(grown.end(), o.emitted.begin(), o.emitted.end());
            flat.insert(flat.end(), o.emitted.begin(), o.emitted.end());
            rows.insert(rows.end(), o.probs.begin(), o.probs.end());
            rs.push_back(dbl_retrieval_result{o.matched_len, static_cast<int>(o.emitted.size()), o.source, o.n_probs});
        }
        if (static_cast<int>(flat.size()) > tokens_cap) dbl::throw_invalid("token buffer too small");
        if (probs && static_cast<int64_t>(rows.size()) > probs_cap) dbl::throw_invalid("probs buffer too small");
        std::memcpy(tokens, flat.data(), flat.size() * 4);
        if (probs && !rows.empty()) std::memcpy(probs, rows.data(), rows.size() * sizeof(double));
        if (segs) std::memcpy(segs, rs.data(), rs.size() * sizeof(dbl_retrieval_result));
        if (n_tokens) *n_tokens = static_cast<int>(flat.size());
    });
}
int dbl_measure_amt(const int32_t* matched_lens, int n, double* out) {
    return guarded([&] {  // speculation.cpp:88-94
        need(out, "out");
        if (n <= 0) dbl::throw_invalid("measure_amt: empty trace");
        need(matched_lens, "matched lengths");
        double sum = 0.0;
        for (int i = 0; i < n; ++i) sum += matched_lens[i];
        *out = sum / static_cast<double>(n);
    });
}

// --------------------------------------------------------------------- decoder state machine
struct dbl_session_s {
    std::unique_ptr<dbl::RoundSession> impl;
    int device;
};

namespace {
const char* const kModeNames[] = {"pre_verify", "post_verify", "ar", "serial"};
const char* const kKindNames[] = {"pending_reject", "extend_keep_draft", "extend_draft_subsumed",
                                  "extend_drop_draft", "ar_step", "reject", "all_accepted"};
const char* const kSourceNames[] = {"prior", "dynamic", "rejected", "context", "miss"};
int name_index(const char* const* names, int n, const std::string& s) {
    for (int i = 0; i < n; ++i)
        if (s == names[i]) return i;
    dbl::throw_invalid("unknown trace label '" + s + "'");
}
dbl_round_trace to_c(const dbl::Trace& t) {
    dbl_round_trace c{};
    c.round = t.round;
    c.mode = name_index(kModeNames, 4, t.mode);
    c.pending = t.pending;
    c.draft_len = t.draft_len;
    if (t.draft_matched.size() > DBL_MAX_SEGS) dbl::throw_invalid("trace has more than DBL_MAX_SEGS segments");
    c.n_draft_matched = static_cast<int>(t.draft_matched.size());
    for (size_t k = 0; k < t.draft_matched.size(); ++k) c.draft_matched[k] = t.draft_matched[k];
    c.target_matched = t.target_matched;
    c.target_source = t.target_source.empty() ? DBL_SRC_MISS : name_index(kSourceNames, 5, t.target_source);
    c.accepted_pending = t.accepted_pending;
    c.pending_reject = t.pending_reject;
    c.rejected = t.rejected;
    c.committed_count = t.committed_count;
    c.kind = name_index(kKindNames, 7, t.kind);
    c.clock_delta = t.clock_delta;
    return c;
}
std::vector<dbl::Trace> from_c(const dbl_round_trace* ts, int n) {
    std::vector<dbl::Trace> out;
    for (int i = 0; i < n; ++i) {
        const dbl_round_trace& c = ts[i];
        if (c.mode < 0 || c.mode > 3 || c.kind < 0 || c.kind > 6 || c.target_source < 0 || c.target_source > 4 ||
            c.n_draft_matched < 0 || c.n_draft_matched > DBL_MAX_SEGS)
            dbl::throw_invalid("trace field out of range");
        dbl::Trace t;
        t.round = c.round;
        t.mode = kModeNames[c.mode];
        t.pending = c.pending;
        t.draft_len = c.draft_len;
        t.draft_matched.assign(c.draft_matched, c.draft_matched + c.n_draft_matched);
        t.target_matched = c.target_matched;
        t.target_source = kSourceNames[c.target_source];
        t.accepted_pending = c.accepted_pending;
        t.pending_reject = c.pending_reject != 0;
        t.rejected = c.rejected != 0;
        t.committed_count = c.committed_count;
        t.kind = kKindNames[c.kind];
        t.clock_delta = c.clock_delta;
        out.push_back(std::move(t));
    }
    return out;
}
}  // namespace

int dbl_rollback(dbl_pipeline_state* st, int64_t keep_len) {
    return guarded([&] {  // pipeline.cpp:15-30
        need(st, "state");
        const int64_t ctx_len = st->n_committed + st->n_speculative;
        if (keep_len > ctx_len) dbl::throw_invalid("rollback: keep_len beyond context");
        if (keep_len < st->last_committed_len) dbl::throw_logic("rollback: keep_len below committed boundary");
        if (keep_len < st->n_committed) st->n_committed = keep_len;
        st->n_speculative = 0;
        st->n_spec_probs = 0;
        st->mode = 0;
    });
}
int dbl_session_create(dbl_model_t draft, dbl_model_t target, dbl_session_t* out) {
    return guarded([&] {
        need(draft, "draft");
        need(target, "target");
        need(out, "out");
        *out = new dbl_session_s{std::make_unique<dbl::RoundSession>(*draft->impl, *target->impl),
                                 target->impl->device()};
    });
}
int dbl_session_destroy(dbl_session_t s) {
    return guarded([&] { delete s; });
}
int dbl_run_round(dbl_session_t s, dbl_store_t store, const dbl_pipeline_options* opts, dbl_pipeline_state* st,
                  dbl_round_trace* trace) {
    return guarded([&] {
        need(s, "session");
        need(store, "store");
        need(opts, "options");
        need(st, "state");
        if (st->n_committed < 0 || st->n_speculative < 0 || st->n_committed > st->committed_cap ||
            st->n_speculative > st->speculative_cap)
            dbl::throw_invalid("state lengths out of range");
        if (st->n_committed > 0) need(st->committed, "committed");
        if (st->n_speculative > 0) need(st->speculative, "speculative");
        // capacities first: the round mutates the datastore, so it must never fail after it ran
        const int64_t grow = st->n_speculative + opts->depth + 1;
        if (st->committed_cap < st->n_committed + grow)
            dbl::throw_invalid("committed buffer too small (need n_committed + n_speculative + depth + 1)");
        if (st->speculative_cap < static_cast<int64_t>(opts->gamma) * (opts->depth + 1))
            dbl::throw_invalid("speculative buffer too small (need gamma * (depth + 1))");
        if (opts->temperature != 0.0 && st->spec_probs &&
            st->spec_probs_cap < static_cast<int64_t>(opts->gamma) * (opts->depth + 1))
            dbl::throw_invalid("spec_probs buffer too small (need gamma * (depth + 1) rows)");
        dbl::HostPipelineState h;
        h.committed.assign(st->committed, st->committed + st->n_committed);
        h.speculative.assign(st->speculative, st->speculative + st->n_speculative);
        h.n_spec_probs = static_cast<long>(st->n_spec_probs);
        h.spec_probs_in = opts->temperature != 0.0 ? st->spec_probs : nullptr;
        h.mode = st->mode;
        h.prev_tokens = st->prev_tokens;
        h.round = static_cast<long>(st->round);
        h.clock = st->clock;
        h.last_committed_len = static_cast<long>(st->last_committed_len);
        std::vector<double> rows;
        const dbl::Trace t = s->impl->run_round(h, *store->impl, *opts,
                                                opts->temperature != 0.0 && st->spec_probs ? &rows : nullptr);
        std::memcpy(st->committed, h.committed.data(), h.committed.size() * 4);
        st->n_committed = static_cast<int64_t>(h.committed.size());
        if (!h.speculative.empty()) std::memcpy(st->speculative, h.speculative.data(), h.speculative.size() * 4);
        st->n_speculative = static_cast<int64_t>(h.speculative.size());
        st->n_spec_probs = h.n_spec_probs;
        if (!rows.empty()) std::memcpy(st->spec_probs, rows.data(), rows.size() * sizeof(double));
        st->mode = h.mode;
        st->prev_tokens = h.prev_tokens;
        st->round = h.round;
        st->clock = h.clock;
        st->last_committed_len = h.last_committed_len;
        if (trace) *trace = to_c(t);
    });
}
int dbl_compute_metrics(const dbl_round_trace* traces, int n, double t_target, dbl_run_metrics* out) {
    return guarded([&] {
        need(out, "out");
        if (n <= 0) dbl::throw_invalid("compute_metrics: no traces");  // pipeline.cpp:327
        need(traces, "traces");
        *out = dbl_run_metrics{};
        dbl::compute_metrics(from_c(traces, n), t_target, out);
    });
}
int dbl_traces_to_jsonl(const dbl_round_trace* traces, int n, char* buf, int64_t cap, int64_t* len) {
    return guarded([&] {
        if (n < 0) dbl::throw_invalid("negative trace count");
        if (n > 0) need(traces, "traces");
        const std::string js = dbl::traces_to_jsonl(from_c(traces, n));
        if (len) *len = static_cast<int64_t>(js.size());
        if (buf) {
            if (cap < static_cast<int64_t>(js.size()) + 1) dbl::throw_invalid("jsonl buffer too small");
            std::memcpy(buf, js.c_str(), js.size() + 1);
        }
    });
}
int dbl_write_traces(const dbl_round_trace* traces, int n, const char* path) {
    return guarded([&] {
        need(path, "path");
        if (n < 0) dbl::throw_invalid("negative trace count");
        if (n > 0) need(traces, "traces");
        const std::string js = dbl::traces_to_jsonl(from_c(traces, n));
        std::FILE* f = std::fopen(path, "wb");
        if (!f) dbl::throw_runtime(std::string("cannot write ") + path);  // pipeline.cpp:398
        const bool ok = std::fwrite(js.data(), 1, js.size(), f) == js.size();
        std::fclose(f);
        if (!ok) dbl::throw_runtime(std::string("cannot write ") + path);
    });
}
int dbl_last_run_traces(dbl_round_trace* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        if (n) *n = static_cast<int64_t>(g_last_traces.size());
        if (out) {
            if (cap < static_cast<int64_t>(g_last_traces.size())) dbl::throw_invalid("trace buffer too small");
            for (size_t i = 0; i < g_last_traces.size(); ++i) out[i] = to_c(g_last_traces[i]);
        }
    });
}
int dbl_store_clone(dbl_store_t src, dbl_store_t* out) {
    return guarded([&] {
        need(src, "store");
        need(out, "out");
        *out = new dbl_store_s{src->impl->clone()};
    });
}
int dbl_build_prior(dbl_store_t s, const int64_t* seq_off, const int32_t* tokens, int n_seqs, int max_order,
                    int rounds) {
    return guarded([&] {  // datastore.cpp:149-159
        need(s, "store");
        if (rounds < 0) dbl::throw_invalid("build_prior: rounds must be >= 0");
        if (n_seqs < 0) dbl::throw_invalid("negative sequence count");
        const int take = std::min(n_seqs, rounds);
        if (take > 0) {
            need(seq_off, "sequence offsets");
            need(tokens, "tokens");
        }
        s->impl->load_layer(DBL_LAYER_PRIOR, max_order, seq_off, tokens, take, 0);
    });
}

// ------------------------------------------------------------------------------ decode loop
int dbl_run(dbl_model_t draft, dbl_model_t target, dbl_store_t store, const int32_t* prompt, int n_prompt,
            int max_new, const dbl_pipeline_options* opts, int32_t* out, int cap, int* n_out,
            dbl_run_metrics* metrics, char* jsonl, int64_t jsonl_cap, int64_t* jsonl_len) {
    return guarded([&] {
        need(draft, "draft");
        need(target, "target");
        need(store, "store");
        need(opts, "options");
        if (n_prompt > 0) need(prompt, "prompt");
        const dbl::RunOutput r = dbl::run_double(*draft->impl, *target->impl, *store->impl, prompt,
                                                 n_prompt, max_new, *opts);
        g_last_log = r.log;
        copy_run(r, out, cap, n_out, metrics, jsonl, jsonl_cap, jsonl_len);
    });
}
int dbl_last_run_log(int32_t* buf, int64_t cap, int64_t* len) {
    return guarded([&] {
        if (len) *len = static_cast<int64_t>(g_last_log.size());
        if (buf) {
            if (cap < static_cast<int64_t>(g_last_log.size())) dbl::throw_invalid("log buffer too small");
            std::memcpy(buf, g_last_log.data(), g_last_log.size() * 4);
        }
    });
}
int dbl_last_run_jsonl(char* buf, int64_t cap, int64_t* len) {
    return guarded([&] {
        if (len) *len = static_cast<int64_t>(g_last_jsonl.size());
        if (buf) {
            if (cap < static_cast<int64_t>(g_last_jsonl.size()) + 1) dbl::throw_invalid("jsonl buffer too small");
            std::memcpy(buf, g_last_jsonl.c_str(), g_last_jsonl.size() + 1);
        }
    });
}
int dbl_set_exact_sampling(int on) {
    return guarded([&] { dbl::set_exact_sampling(on != 0); });
}

int dbl_run_ar(dbl_model_t target, const int32_t* prompt, int n_prompt, int max_new, double t_target,
               int32_t* out, int cap, int* n_out, dbl_run_metrics* metrics, char* jsonl,
               int64_t jsonl_cap, int64_t* jsonl_len) {
    return guarded([&] {
        need(target, "target");
        if (n_prompt > 0) need(prompt, "prompt");
        const dbl::RunOutput r = dbl::run_ar(*target->impl, prompt, n_prompt, max_new, t_target, 0.0, 0);
        copy_run(r, out, cap, n_out, metrics, jsonl, jsonl_cap, jsonl_len);
    });
}
int dbl_run_ar_sampled(dbl_model_t target, const int32_t* prompt, int n_prompt, int max_new, double t_target,
                       double temperature, uint64_t seed, int32_t* out, int cap, int* n_out,
                       dbl_run_metrics* metrics, char* jsonl, int64_t jsonl_cap, int64_t* jsonl_len) {
    return guarded([&] {
        need(target, "target");
        if (n_prompt > 0) need(prompt, "prompt");
        const dbl::RunOutput r =
            dbl::run_ar(*target->impl, prompt, n_prompt, max_new, t_target, temperature, seed);
        copy_run(r, out, cap, n_out, metrics, jsonl, jsonl_cap, jsonl_len);
    });
}
int dbl_run_batch(dbl_model_t draft, dbl_model_t target, int n_seq, const dbl_store_t* stores,
                  const int64_t* prompt_off, const int32_t* prompt_tokens, int max_new,
                  const dbl_pipeline_options* opts, int32_t* out, int32_t* out_n, dbl_run_metrics* metrics,
                  char* jsonl, int64_t jsonl_cap, int64_t* jsonl_lens) {
    return guarded([&] {
        need(draft, "draft");
        need(target, "target");
        need(stores, "stores");
        need(prompt_off, "prompt_off");
        need(prompt_tokens, "prompt_tokens");
        need(opts, "options");
        need(out, "out");
        need(out_n, "out_n");
        if (n_seq < 1) dbl::throw_invalid("n_seq must be >= 1");
        std::vector<dbl::DeviceStore*> sts(n_seq);
        std::vector<std::vector<int32_t>> prompts(n_seq);
        for (int b = 0; b < n_seq; ++b) {
            need(stores[b], "store");
            sts[b] = stores[b]->impl.get();
            if (prompt_off[b + 1] < prompt_off[b]) dbl::throw_invalid("prompt offsets must be non-decreasing");
            prompts[b].assign(prompt_tokens + prompt_off[b], prompt_tokens + prompt_off[b + 1]);
        }
        const auto res = dbl::run_double_multi(*draft->impl, *target->impl, sts, prompts, max_new, *opts);
        int64_t at = 0;
        for (int b = 0; b < n_seq; ++b) {
            copy_run(res[b], out + static_cast<size_t>(b) * max_new, max_new, nullptr, metrics ? metrics + b : nullptr,
                     nullptr, 0, nullptr);
            out_n[b] = static_cast<int32_t>(res[b].output.size());
            if (jsonl || jsonl_lens) {
                const std::string js = dbl::traces_to_jsonl(res[b].traces);
                if (jsonl_lens) jsonl_lens[b] = static_cast<int64_t>(js.size());
                if (jsonl) {
                    if (at + static_cast<int64_t>(js.size()) + 1 > jsonl_cap) dbl::throw_invalid("jsonl buffer too small");
                    std::memcpy(jsonl + at, js.data(), js.size());
                    at += static_cast<int64_t>(js.size());
                    jsonl[at] = 0;
                }
            }
        }
    });
}
int dbl_run_ar_batch(dbl_model_t target, int n_seq, const int64_t* prompt_off, const int32_t* prompt_tokens,
                     int max_new, int32_t* out, int32_t* out_n, double* device_ms, int64_t* kernel_launches) {
    return guarded([&] {
        need(target, "target");
        need(prompt_off, "prompt_off");
        need(prompt_tokens, "prompt_tokens");
        need(out, "out");
        need(out_n, "out_n");
        if (n_seq < 1) dbl::throw_invalid("n_seq must be >= 1");
        std::vector<std::vector<int32_t>> prompts(n_seq);
        for (int b = 0; b < n_seq; ++b) {
            if (prompt_off[b + 1] < prompt_off[b]) dbl::throw_invalid("prompt offsets must be non-decreasing");
            prompts[b].assign(prompt_tokens + prompt_off[b], prompt_tokens + prompt_off[b + 1]);
        }
        double ms = 0.0;
        long long launches = 0;
        const auto res = dbl::run_ar_batch(*target->impl, prompts, max_new, 1.0, &ms, &launches);
        for (int b = 0; b < n_seq; ++b) {
            out_n[b] = static_cast<int32_t>(res[b].output.size());
            std::memcpy(out + static_cast<size_t>(b) * max_new, res[b].output.data(), res[b].output.size() * 4);
        }
        if (device_ms) *device_ms = ms;
        if (kernel_launches) *kernel_launches = launches;
    });
}
int dbl_run_serial_sd(dbl_model_t draft, dbl_model_t target, dbl_store_t store, const int32_t* prompt,
                      int n_prompt, int max_new, const dbl_pipeline_options* opts, int use_retrieval,
                      int32_t* out, int cap, int* n_out, dbl_run_metrics* metrics, char* jsonl,
                      int64_t jsonl_cap, int64_t* jsonl_len) {
    return guarded([&] {
        need(draft, "draft");
        need(target, "target");
        need(store, "store");
        need(opts, "options");
        if (n_prompt > 0) need(prompt, "prompt");
        const dbl::RunOutput r = dbl::run_serial_sd(*draft->impl, *target->impl, *store->impl, prompt,
                                                    n_prompt, max_new, *opts, use_retrieval != 0);
        copy_run(r, out, cap, n_out, metrics, jsonl, jsonl_cap, jsonl_len);
    });
}

int dbl_profile_forward(dbl_model_t m, int ctx_len, int rows, int iters, double* out) {
    return guarded([&] {
        need(m, "model");
        need(out, "out");
        dbl::profile_forward(*m->impl, ctx_len, rows, iters, out);
    });
}

// Back-to-back launches of one GEMM shape (weights/activations resident): ms per launch.  With
// `chain` > 1 the weights rotate over `chain` distinct copies (no L2 reuse between launches).
int dbl_debug_gemm_bench(int epi, int n_out, int K, int tp, int iters, int chain, double* ms_per_launch) {
    return guarded([&] {
        using namespace dbl;
        require_device(0);
        chain = std::max(chain, 1);
        std::vector<DevBuf<__nv_bfloat16>> W(chain);
        std::vector<CUtensorMap> tW(chain);
        for (int i = 0; i < chain; ++i) {
            W[i].alloc(static_cast<size_t>(n_out) * K);
            launch_init_normal(W[i].p, n_out, K, K, 7 + i, 1, 0, 0, K, 0.02f, 0);
            tW[i] = make_tmap_bf16_2d(W[i].p, n_out, K, 128);
        }
        DevBuf<__nv_bfloat16> X(static_cast<size_t>(tp) * K);
        launch_init_normal(X.p, tp, K, K, 3, 2, 0, 0, K, 1.0f, 0);
        const CUtensorMap tX = make_tmap_bf16_2d(X.p, tp, K, 16);
        GemmWorkspace ws;
        ws.ensure(num_sms(0), tp, (n_out + 127) / 128);
        const int cols = epi == 2 ? n_out / 2 : n_out;
        DevBuf<float> o32(static_cast<size_t>(tp) * cols);
        DevBuf<__nv_bfloat16> o16(static_cast<size_t>(tp) * cols);
        o32.zero();
        void* out = (epi == 0 || epi == 2) ? static_cast<void*>(o16.p) : static_cast<void*>(o32.p);
        cudaStream_t s;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        for (int i = 0; i < 3; ++i)
            gemm_launch(static_cast<Epi>(epi), tW[i % chain], tX, n_out, K, tp, n_out, out, cols, nullptr, 0, ws, s);
        cudaEvent_t a, b;
        CUDA_CHECK(cudaEventCreate(&a));
        CUDA_CHECK(cudaEventCreate(&b));
        CUDA_CHECK(cudaEventRecord(a, s));
        for (int i = 0; i < iters; ++i)
            gemm_launch(static_cast<Epi>(epi), tW[i % chain], tX, n_out, K, tp, n_out, out, cols, nullptr, 0, ws, s);
        CUDA_CHECK(cudaEventRecord(b, s));
        CUDA_CHECK(cudaStreamSynchronize(s));
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        *ms_per_launch = ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(s);
    });
}

// GEMM timeline (DBL_GEMM_TRACE=1): stamps [n_launches][kTraceCtas][4], grids, weight bytes
int dbl_debug_gemm_trace(uint64_t* stamps, int64_t cap, int32_t* grids, int64_t* bytes, int* n_launches) {
    return guarded([&] {
        dbl::GemmTrace& t = dbl::gemm_trace();
        *n_launches = t.n;
        const int64_t need = static_cast<int64_t>(t.n) * dbl::kTraceCtas * 4;
        if (t.n == 0) return;
        if (cap < need) dbl::throw_invalid("trace buffer too small");
        CUDA_CHECK(cudaDeviceSynchronize());
        CUDA_CHECK(cudaMemcpy(stamps, t.buf.p, need * 8, cudaMemcpyDeviceToHost));
        for (int i = 0; i < t.n; ++i) {
            grids[i] = t.grid[i];
            bytes[i] = t.bytes[i];
        }
        t.n = 0;
        t.grid.clear();
        t.bytes.clear();
    });
}

// --------------------------------------------------------------------------- kernel checks
// ------------------------------------------------------------------------ verifier + RNG

int dbl_rng_create(uint64_t seed, int device, dbl_rng_t* out) {
    return guarded([&] {
        need(out, "out");
        *out = new dbl_rng_s{std::make_unique<dbl::DeviceRng>(seed, device)};
    });
}
int dbl_rng_derive(uint64_t seed, uint64_t round, uint64_t lane, int device, dbl_rng_t* out) {
    return guarded([&] {
        need(out, "out");
        *out = new dbl_rng_s{std::make_unique<dbl::DeviceRng>(dbl::DeviceRng::derive(seed, round, lane, device))};
    });
}
int dbl_rng_uniform(dbl_rng_t r, double* out, int n) {
    return guarded([&] {
        need(r, "rng");
        r->impl->uniform(out, n);
    });
}
int dbl_rng_destroy(dbl_rng_t r) {
    return guarded([&] { delete r; });
}
int dbl_accept_prob(const double* p, int np, const double* q, int nq, int32_t x, double* out) {
    return guarded([&] {
        need(p, "p");
        need(q, "q");
        need(out, "out");
        *out = dbl::accept_prob(p, np, q, nq, x, 0);
    });
}
int dbl_residual_sample(const double* p, int np, const double* q, int nq, dbl_rng_t r, int32_t* out) {
    return guarded([&] {
        need(p, "p");
        need(q, "q");
        need(r, "rng");
        need(out, "out");
        *out = dbl::residual_sample(p, np, q, nq, *r->impl);
    });
}
int dbl_residual_sample_point_mass(const double* p, int np, int32_t x, dbl_rng_t r, int32_t* out) {
    return guarded([&] {
        need(p, "p");
        need(r, "rng");
        need(out, "out");
        *out = dbl::residual_sample_point_mass(p, np, x, *r->impl);
    });
}
int dbl_verify_against_target(const int32_t* draft, int n_draft, const double* draft_probs, const int64_t* draft_off,
                              int n_draft_rows, const double* target_probs, const int64_t* target_off,
                              int n_target_rows, double temperature, dbl_rng_t r, int* first_reject) {
    return guarded([&] {
        need(r, "rng");
        need(first_reject, "first_reject");
        *first_reject = dbl::verify_against_target(draft, n_draft, draft_probs, draft_off, n_draft_rows, target_probs,
                                                   target_off, n_target_rows, temperature, *r->impl);
    });
}
int dbl_guided_output(const int32_t* draft, int n_draft, const double* draft_probs, const int64_t* draft_off,
                      int n_draft_rows, const int32_t* guide_tokens, int n_guide, const double* guide_probs,
                      const int64_t* guide_off, int n_guide_rows, int first_reject, double temperature, dbl_rng_t r,
                      int32_t* committed, int cap, int* n_committed, int* accepted_len, int* kind) {
    return guarded([&] {
        need(r, "rng");
        need(n_committed, "n_committed");
        need(accepted_len, "accepted_len");
        need(kind, "kind");
        const dbl::VerifyOutcome o =
            dbl::guided_output(draft, n_draft, draft_probs, draft_off, n_draft_rows, guide_tokens, n_guide,
                               guide_probs, guide_off, n_guide_rows, first_reject, temperature, *r->impl);
        *n_committed = static_cast<int>(o.committed.size());
        *accepted_len = o.accepted_len;
        *kind = o.kind;
        if (static_cast<int>(o.committed.size()) > cap) dbl::throw_invalid("committed buffer too small");
        if (!o.committed.empty()) {
            need(committed, "committed");
            std::memcpy(committed, o.committed.data(), o.committed.size() * 4);
        }
    });
}

int dbl_debug_fwd_trace(uint64_t* stamps, int64_t cap, int* n_ph, int* grid) {
    return guarded([&] {
        need(n_ph, "n_ph");
        need(grid, "grid");
        dbl::fwd_trace_read(reinterpret_cast<unsigned long long*>(stamps), cap, n_ph, grid);
    });
}

int dbl_debug_gemm(int epi, const uint16_t* W, int n_out, int K, const uint16_t* X, int T, int tp,
                   int n_valid, float* io, int32_t* argmax) {
    return guarded([&] {
        need(W, "W");
        need(X, "X");
        if (T < 1 || T > tp) dbl::throw_invalid("need 1 <= T <= tp");
        dbl::require_device(0);
        using namespace dbl;
        DevBuf<uint16_t> dW(static_cast<size_t>(n_out) * K), dX(static_cast<size_t>(tp) * K);
        CUDA_CHECK(cudaMemcpy(dW.p, W, dW.bytes(), cudaMemcpyHostToDevice));
        dX.zero();
        CUDA_CHECK(cudaMemcpy(dX.p, X, static_cast<size_t>(T) * K * 2, cudaMemcpyHostToDevice));
        const CUtensorMap tW = make_tmap_bf16_2d(dW.p, n_out, K, 128);
        const CUtensorMap tX = make_tmap_bf16_2d(dX.p, tp, K, 16);
        GemmWorkspace ws;
        const int n_tiles = (n_out + 127) / 128;
        ws.ensure(num_sms(0), tp, n_tiles);
        const int out_cols = epi == 2 ? n_out / 2 : n_out;
        DevBuf<float> o32(static_cast<size_t>(tp) * out_cols);
        DevBuf<__nv_bfloat16> o16(static_cast<size_t>(tp) * out_cols);
        o32.zero();
        if (epi == 1) CUDA_CHECK(cudaMemcpy(o32.p, io, static_cast<size_t>(T) * out_cols * 4, cudaMemcpyHostToDevice));
        void* out = (epi == 0 || epi == 2) ? static_cast<void*>(o16.p) : static_cast<void*>(o32.p);
        gemm_launch(static_cast<Epi>(epi), tW, tX, n_out, K, tp, n_valid, out, out_cols,
                    epi == 3 ? o32.p : nullptr, out_cols, ws, 0);
        if (epi == 3) {
            LaneState st{};
            st.L = T; st.c = 0; st.start = 0;
            LaneState* dst = nullptr;
            CUDA_CHECK(cudaMalloc(&dst, sizeof st));
            CUDA_CHECK(cudaMemcpy(dst, &st, sizeof st, cudaMemcpyHostToDevice));
            DevBuf<int32_t> am(tp);
            argmax_finish(ws, n_tiles, tp, dst, am.p, 0);
            CUDA_CHECK(cudaMemcpy(argmax, am.p, T * 4, cudaMemcpyDeviceToHost));
            cudaFree(dst);
        }
        CUDA_CHECK(cudaDeviceSynchronize());
        if (epi == 0 || epi == 2) {
            std::vector<__nv_bfloat16> h(static_cast<size_t>(T) * out_cols);
            CUDA_CHECK(cudaMemcpy(h.data(), o16.p, h.size() * 2, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < h.size(); ++i) io[i] = __bfloat162float(h[i]);
        } else {
            CUDA_CHECK(cudaMemcpy(io, o32.p, static_cast<size_t>(T) * out_cols * 4, cudaMemcpyDeviceToHost));
        }
    });
}

}  // extern "C"
