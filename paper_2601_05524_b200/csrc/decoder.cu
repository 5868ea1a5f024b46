// The DOUBLE decode loop, B200 edition.
//
// Per round (run_round, pipeline.cpp:223-262) the draft and target lanes run concurrently on two
// CUDA streams over the same frozen datastore snapshot (the reference's Engine::Concurrent contract,
// pipeline.cpp:239-261):
//   draft stream : gamma x [lookup -> draft forward -> accept]  (no host round trip inside the chain)
//   target stream: lookup -> ONE verify forward over committed[kv..] ⊕ spec ⊕ cands -> accept/pre-verify
// Both write their results into mapped pinned memory; the host joins, applies finish_round
// (pipeline.cpp:91-206) exactly as the reference, enqueues the <= 3 datastore appends and the lane
// cursor updates, and starts the next round.  KV "rollback" is a length update: kv_len := LCP of what
// the device processed and the new committed ⊕ speculative context.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "accept.cuh"
#include "decoder.cuh"
#include "rng.cuh"
#include "sampling.cuh"

namespace dbl {

// ------------------------------------------------------------------------------------ Lane
namespace {
__global__ void set_lane_state_kernel(LaneState* st, int L, int c, int kv, int row0) {
    st->L = L;
    st->c = c;
    st->kv_len = kv;
    st->row0 = row0;
    st->src = DBL_SRC_MISS;
    st->order = 0;
    st->start = min(kv, row0);
}
}  // namespace

Lane::Lane(Model& m, int cap) : model(m), capacity(cap) {
    DeviceGuard g(m.device());
    buf.alloc(cap);
    argmax.alloc(cap);
    buf.zero();
    CUDA_CHECK(cudaMalloc(&state, sizeof(LaneState)));
    CUDA_CHECK(cudaMemsetAsync(state, 0, sizeof(LaneState), 0));
    // complete before the lane is used: its token uploads and kernels run on non-blocking streams that
    // do not order after the legacy stream (an in-flight memset here once zeroed uploaded tokens)
    CUDA_CHECK(cudaStreamSynchronize(0));
    cache = m.make_cache(cap);
}
Lane::~Lane() {
    if (state) cudaFree(state);
    if (cache) model.recycle_cache(std::move(cache));
}
void Model::forward_lanes(const std::vector<Lane*>& lanes, int max_tokens, cudaStream_t s) {
    for (Lane* l : lanes) forward(*l, max_tokens, s);  // stateless models: one forward per lane
}

void Lane::set_state(int L, int c, int kv, int row0, cudaStream_t s) {
    set_lane_state_kernel<<<1, 1, 0, s>>>(state, L, c, kv, row0);
    CUDA_LAUNCH_CHECK();
}

namespace {

// pinned mirror used to upload lane tokens: stage[pos] == token at pos
struct LaneIO {
    Lane* lane;
    PinBuf<int32_t> stage;
    explicit LaneIO(Lane* l) : lane(l), stage(l->capacity) {}
    // make the device buffer hold X in [0, |X|) given the mirror; returns the LCP
    int sync_tokens(const std::vector<int32_t>& X, cudaStream_t s) {
        if (static_cast<int>(X.size()) > lane->capacity) throw_runtime("lane capacity exceeded");
        const auto& mi = lane->mirror;
        size_t l = 0;
        const size_t lim = std::min(mi.size(), X.size());
        while (l < lim && mi[l] == X[l]) ++l;
        if (l < X.size()) {
            std::memcpy(stage.p + l, X.data() + l, (X.size() - l) * 4);
            CUDA_CHECK(cudaMemcpyAsync(lane->buf.p + l, stage.p + l, (X.size() - l) * 4,
                                       cudaMemcpyHostToDevice, s));
        }
        lane->mirror = X;
        return static_cast<int>(l);
    }
};

constexpr int kPrefillChunkMax = 256;
// DBL_PREFILL_CHUNK (experiments): a smaller prefill / long-forward piece
const int kPrefillChunk = [] {
    const char* e = std::getenv("DBL_PREFILL_CHUNK");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 && v <= kPrefillChunkMax ? v : kPrefillChunkMax;
}();

// advance the lane's KV to `upto` (positions [kv_len, upto) processed), in forward-sized chunks
void catch_up(Lane& lane, int upto, cudaStream_t s) {
    if (!lane.model.has_kv()) return;
    const int chunk = std::min(kPrefillChunk, lane.model.max_forward_tokens());
    while (lane.kv_len < upto) {
        const int end = std::min(upto, lane.kv_len + chunk);
        // process [kv_len, end): L = end, c = 0, row0 = end - 1 >= kv_len
        lane.set_state(end, 0, lane.kv_len, end - 1, s);
        lane.model.forward(lane, end - lane.kv_len, s);
        lane.kv_len = end;
    }
}

// forward_batch has no row cap (model.cpp:37-53), one device forward carries <= 256 token columns.  A
// longer forward (a verify over a gamma >= ~23 speculative tail, or a draft segment after a long
// commit) is split: positions [first, e) — KV and argmax rows — are processed first in <= 256-row
// chunks, so the forward issued next covers [e, L + c_max) only.  Batch invariance makes every row
// bitwise the row of the unsplit forward.  Must run before the lane's lookup (set_state resets it).
// Returns the first position the next forward processes (its row bound is L + c_max - that).
int split_long_forward(Lane& lane, int L, int row0, int c_max, bool sampled, cudaStream_t s) {
    const int first = std::min(lane.kv_len, row0);
    if (!lane.model.has_kv()) return first;
    const int cap = std::min(kPrefillChunk, lane.model.max_forward_tokens());
    if (L + c_max - first <= cap) return first;
    if (sampled) throw_runtime("sampled forward exceeds 256 consumed rows (gamma * (depth + 1) too large)");
    const int e = L + c_max - cap;
    lane.kv_len = first;  // [first, kv_len) is recomputed with its rows (identical KV rewritten)
    catch_up(lane, e, s);
    lane.set_state(L, 0, e, e, s);
    return e;
}

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    Timer() {
        CUDA_CHECK(cudaEventCreate(&a));
        CUDA_CHECK(cudaEventCreate(&b));
    }
    ~Timer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    float ms() const {
        float m = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&m, a, b));
        return m;
    }
};

// The round's streams.  Target side (verify forward, finish_round's datastore appends, the target
// lane): `main` + `target` on the target's device.  Draft side: `draft` (+ `dmain` for its lane and
// datastore-mirror updates) on the draft's device — the same device (dmain aliases main) or its own
// GPU (PSD draft-while-verify across devices: the host joins both sides at the round boundary).
struct Streams {
    cudaStream_t main = nullptr, draft = nullptr, target = nullptr, dmain = nullptr;
    cudaEvent_t ready = nullptr, tf0 = nullptr, tf1 = nullptr;
    cudaEvent_t dready = nullptr;  // on the draft's device (events record only on their own device)
    int tdev = 0, ddev = 0;
    Streams() : Streams(current_device(), current_device()) {}
    Streams(int target_dev, int draft_dev) : tdev(target_dev), ddev(draft_dev) {
        // The target's verify forward is the round's critical path: its stream gets the highest
        // priority so a co-located draft chain fills SM gaps instead of delaying target CTAs.
        int lo = 0, hi = 0;
        {
            DeviceGuard g(tdev);
            CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CUDA_CHECK(cudaStreamCreateWithPriority(&main, cudaStreamNonBlocking, hi));
            CUDA_CHECK(cudaStreamCreateWithPriority(&target, cudaStreamNonBlocking, hi));
            own_target = target;
            CUDA_CHECK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
            CUDA_CHECK(cudaEventCreate(&tf0));
            CUDA_CHECK(cudaEventCreate(&tf1));
            // The API's store / model calls run on the legacy stream and are asynchronous; these streams
            // are non-blocking, so order the loop after everything already enqueued there (e.g. the
            // prior's inserts of build_prior) explicitly.
            CUDA_CHECK(cudaEventRecord(ready, 0));
            CUDA_CHECK(cudaStreamWaitEvent(main, ready, 0));
        }
        DeviceGuard g(ddev);
        CUDA_CHECK(cudaStreamCreateWithPriority(&draft, cudaStreamNonBlocking, lo));
        CUDA_CHECK(cudaEventCreateWithFlags(&dready, cudaEventDisableTiming));
        if (ddev != tdev) {
            CUDA_CHECK(cudaStreamCreateWithPriority(&dmain, cudaStreamNonBlocking, hi));
            CUDA_CHECK(cudaEventRecord(dready, 0));
            CUDA_CHECK(cudaStreamWaitEvent(dmain, dready, 0));
        } else {
            dmain = main;
        }
    }
    cudaStream_t own_target = nullptr;  // target may alias draft (see DoubleEngine)
    ~Streams() {
        cudaStreamSynchronize(main);
        cudaStreamSynchronize(draft);
        cudaStreamSynchronize(own_target);
        if (dmain != main) cudaStreamSynchronize(dmain);
        cudaStreamDestroy(main);
        cudaStreamDestroy(draft);
        cudaStreamDestroy(own_target);
        if (dmain != main) cudaStreamDestroy(dmain);
        cudaEventDestroy(ready);
        cudaEventDestroy(dready);
        cudaEventDestroy(tf0);
        cudaEventDestroy(tf1);
    }
    static int current_device() {
        int d = 0;
        CUDA_CHECK(cudaGetDevice(&d));
        return d;
    }
    void fork() {  // each side starts after everything enqueued on its own main stream
        CUDA_CHECK(cudaEventRecord(ready, main));
        CUDA_CHECK(cudaStreamWaitEvent(target, ready, 0));
        if (dmain == main) {
            CUDA_CHECK(cudaStreamWaitEvent(draft, ready, 0));
        } else {
            DeviceGuard g(ddev);
            CUDA_CHECK(cudaEventRecord(dready, dmain));
            CUDA_CHECK(cudaStreamWaitEvent(draft, dready, 0));
        }
    }
    void join_draft_into_main() {  // main (target device) waits for the draft stream's work
        if (dmain == main) {
            CUDA_CHECK(cudaEventRecord(ready, draft));
            CUDA_CHECK(cudaStreamWaitEvent(main, ready, 0));
        } else {
            {
                DeviceGuard g(ddev);
                CUDA_CHECK(cudaEventRecord(dready, draft));
            }
            CUDA_CHECK(cudaStreamWaitEvent(main, dready, 0));
        }
    }
};

const char* source_name(int s) {  // to_string(LookupSource), datastore.cpp:33-42
    static const char* n[] = {"prior", "dynamic", "rejected", "context", "miss"};
    return (s >= 0 && s <= 4) ? n[s] : "?";
}

void validate_opts(const dbl_pipeline_options& o) {  // pipeline.cpp:267-272, pipeline.hpp:24-28
    if (o.gamma < 1) throw_invalid("gamma must be >= 1");
    if (o.depth < 1) throw_invalid("depth must be >= 1");
    // the round record holds <= kMaxRoundTokens target candidates + the continuation (RoundResult)
    if (o.depth > kMaxRoundTokens - 1) throw_invalid("depth must be <= " + std::to_string(kMaxRoundTokens - 1));
    if (o.gamma > kMaxSegs) throw_invalid("gamma exceeds the device chain record");
    if (o.t_target < 0.0 || o.t_draft <= 0.0 || o.t_lookup < 0.0 || o.t_sync < 0.0)
        throw_invalid("latency values out of range");
    if (!(o.temperature >= 0.0)) throw_invalid("temperature must be >= 0");  // harness.cpp:50
}

// Device buffers of the sampled (temperature > 0) loop: the per-round RNG lanes, the draft's and
// target's fp64 distribution rows, and the draft chain's eff rows (double-buffered: the rows kept as
// the next round's spec_probs, pipeline.cpp:166-169, stay readable while the next chain is drafted).
struct Sampled {
    double T;
    uint64_t seed;
    size_t V;
    int chain_rows;
    DevBuf<DevRng> rng;  // rng_d, rng_t, rng_v (run_round, pipeline.cpp:227-231)
    DevBuf<double> ddist, tdist, chain[2], dscratch, tscratch;
    int cur = 0;
    const double* spec_probs = nullptr;
    Sampled(double temp, uint64_t sd, int vocab, int draft_rows, int chain_rows_, int target_rows)
        : T(temp), seed(sd), V(static_cast<size_t>(vocab)), chain_rows(chain_rows_) {
        rng.alloc(3);
        ddist.alloc(V * std::max(draft_rows, 1));
        tdist.alloc(V * std::max(target_rows, 1));
        for (auto& c : chain) c.alloc(V * std::max(chain_rows, 1));
        dscratch.alloc(V);
        tscratch.alloc(3 * V);
    }
};

void check_round_errors(const RoundResult* rr) {
    if (rr->draft_error) raise_sample_error(rr->draft_error);
    if (rr->target_error) raise_sample_error(rr->target_error);
}

// record_accepted_run / record_rejected_run (pipeline.cpp:72-89)
void record_run(DeviceStore& st, int layer, const std::vector<int32_t>& before, const int32_t* add,
                size_t na, cudaStream_t s) {
    if (na == 0) return;
    const size_t pre = std::min<size_t>(layer == 1 ? static_cast<size_t>(st.max_order()) - 1 : 3,
                                        before.size());
    std::vector<int32_t> rec(before.end() - static_cast<long>(pre), before.end());
    rec.insert(rec.end(), add, add + na);
    st.record(layer, rec.data(), static_cast<int>(rec.size()), s);
}

void device_counts(DeviceStore& st, cudaStream_t s, long* lookups, long* hits) {
    int64_t v[6];
    st.stats(v, s);
    *lookups = v[0];
    *hits = v[1] + v[2] + v[3] + v[4];
}

void finish_output(const std::vector<int32_t>& committed, size_t n_prompt, int max_new,
                   RunOutput& r) {
    r.output.assign(committed.begin() + static_cast<long>(n_prompt), committed.end());
    if (r.output.size() > static_cast<size_t>(max_new)) r.output.resize(max_new);
}

}  // namespace

// ------------------------------------------------------------------------------ metrics / jsonl
void compute_metrics(const std::vector<Trace>& traces, double t_target, dbl_run_metrics* m) {
    // compute_metrics, pipeline.cpp:325-371
    long tokens = 0, cur = 0, matched_sum = 0, matched_n = 0, seg_total = 0, seg_n = 0;
    double clock = 0.0;
    for (const Trace& t : traces) {
        tokens += t.committed_count;
        clock += t.clock_delta;
        if (t.pending_reject) {
            seg_total += cur + t.accepted_pending;
            ++seg_n;
            cur = t.committed_count - t.accepted_pending;
        } else if (t.rejected) {
            seg_total += cur + t.committed_count;
            ++seg_n;
            cur = 0;
        } else {
            cur += t.committed_count;
        }
        for (int v : t.draft_matched) { matched_sum += v; ++matched_n; }
        if (t.target_matched >= 0) { matched_sum += t.target_matched; ++matched_n; }
    }
    if (cur > 0) { seg_total += cur; ++seg_n; }
    m->tokens = tokens;
    m->rounds = static_cast<int64_t>(traces.size());
    m->clock = clock;
    m->m = seg_n ? static_cast<double>(seg_total) / static_cast<double>(seg_n) : 0.0;
    m->amt = matched_n ? static_cast<double>(matched_sum) / static_cast<double>(matched_n) : 0.0;
    m->speedup = clock > 0.0 ? static_cast<double>(tokens) * t_target / clock : 0.0;
    m->hit_rate = 0.0;
    m->lookups = 0;
}

namespace {
// nlohmann::json's double rendering (shortest round-trip digits; fixed notation for decimal
// exponents in (-4, 15], else d.ddde+XX; always a '.' or 'e')
std::string json_double(double x) {
    if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
    char tmp[64];
    int prec = 1;
    for (; prec <= 17; ++prec) {
        std::snprintf(tmp, sizeof tmp, "%.*e", prec - 1, x);
        if (std::strtod(tmp, nullptr) == x) break;
    }
    std::string s(tmp);
    bool neg = false;
    size_t i = 0;
    if (s[0] == '-') { neg = true; i = 1; }
    std::string digits;
    for (; i < s.size() && s[i] != 'e'; ++i)
        if (s[i] != '.') digits += s[i];
    const int e10 = std::atoi(s.c_str() + i + 1);
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = static_cast<int>(digits.size()), n = e10 + 1;
    std::string out = neg ? "-" : "";
    if (k <= n && n <= 15) {
        out += digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(-n, '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}
}  // namespace

std::string traces_to_jsonl(const std::vector<Trace>& traces) {  // pipeline.cpp:373-394
    std::string out;
    for (const Trace& t : traces) {
        out += "{\"round\":" + std::to_string(t.round);
        out += ",\"mode\":\"" + t.mode + "\"";
        out += ",\"pending\":" + std::to_string(t.pending);
        out += ",\"draft_len\":" + std::to_string(t.draft_len);
        out += ",\"draft_matched\":[";
        for (size_t k = 0; k < t.draft_matched.size(); ++k) {
            if (k) out += ",";
            out += std::to_string(t.draft_matched[k]);
        }
        out += "],\"target_matched\":" + std::to_string(t.target_matched);
        out += ",\"target_source\":\"" + t.target_source + "\"";
        out += ",\"accepted_pending\":" + std::to_string(t.accepted_pending);
        out += std::string(",\"pending_reject\":") + (t.pending_reject ? "true" : "false");
        out += std::string(",\"rejected\":") + (t.rejected ? "true" : "false");
        out += ",\"committed\":" + std::to_string(t.committed_count);
        out += ",\"kind\":\"" + t.kind + "\"";
        out += ",\"clock_delta\":" + json_double(t.clock_delta) + "}\n";
    }
    return out;
}

// ------------------------------------------------------------------------------- run (DOUBLE)
namespace {
// One sequence of a (possibly batched) DOUBLE decode: PipelineState (pipeline.hpp:46-55), its lanes,
// its datastore and its round record.
struct DoubleSeq {
    DeviceStore* st = nullptr;
    // the draft side's datastore: `st` itself, or (draft on another GPU) a replica on the draft's
    // device that receives the same appends in the same order (SURVEY §8(b) threading: "inserts are
    // applied at the boundary in identical order on every device mirror")
    DeviceStore* dst = nullptr;
    std::unique_ptr<DeviceStore> mirror;
    int64_t mirror_base[6] = {};
    std::unique_ptr<Lane> dl, tl;
    std::unique_ptr<LaneIO> dio, tio;
    PinBuf<RoundResult> rr_buf;
    RoundResult* rr = nullptr;
    RoundResult* rr_dev = nullptr;
    std::unique_ptr<Sampled> smp;
    std::vector<int32_t> committed, spec;
    int n_prompt = 0, mode = 0, prev_tokens = 0;
    long round = 0, last_committed_len = 0;
    size_t scanned = 0;
    bool done = false;
    long base_lookups = 0, base_hits = 0;
    int L = 0, nc = 0, ns = 0;  // this round
    int64_t trows = 0;
    RunOutput res;
};

// The round engine shared by run() (pipeline.cpp:264-323) and the run_round session (pipeline.cpp:
// 223-262): the draft worker (iterative_draft) and the target worker (lookup + one verify forward)
// on two streams over the frozen datastore snapshot, then finish_round (pipeline.cpp:91-206) on the
// host with the datastore appends and the lanes' KV commit enqueued for the next round.
struct DoubleEngine {
    Model& dm;
    Model& tm;
    Streams S;
    double tfwd_ms = 0.0;
    int64_t tfwd_n = 0;

    DoubleEngine(Model& d, Model& t) : dm(d), tm(t), S(t.device(), d.device()) {
        // draft and target run concurrently unless that would put more than two persistent forwards on
        // the draft's GPU (tensor-parallel shards sharing it): then both workers share one stream — the
        // round's results are identical either way (frozen snapshot, pipeline.cpp:239-261)
        if (dm.device() == tm.device() && dm.persistent_grids() + tm.persistent_grids_on(dm.device()) > 2)
            S.target = S.draft;
        if (dm.device() != tm.device() && tm.persistent_grids_on(dm.device()) > 1)
            throw_invalid("draft GPU hosts more than one target shard (at most two persistent forwards per GPU)");
        // shared memory: the draft's and the target's forward CTAs co-reside on every SM of a shared GPU
        if (&dm == &tm) {
            dm.set_smem_budget(kFwdSmemSharedBudget);
        } else if (tm.persistent_grids_on(dm.device()) > 0) {
            dm.set_smem_budget(kFwdSmemDraftBudget);
            tm.set_smem_budget(kFwdSmemBudget);
            colocated_ = true;
        }
    }
    // The driver runs cooperative grids one at a time, so a co-located draft's forward and the verify
    // forward would serialize (§7a).  A draft forward on half the SMs, launched plainly, runs beside the
    // verify's grid (both always fit: 136 + 90 KB, 64 K registers per SM) — worth it while the draft
    // chain fits under the verify (gamma <= 2: 150 -> 170 tok/s on configs[1]); longer chains keep the
    // draft's full grid (each segment is then on the critical path).  DBL_DRAFT_GRID_DIV overrides.
    void configure_draft(int gamma) {
        if (!colocated_) return;
        static const int env = [] {
            const char* e = std::getenv("DBL_DRAFT_GRID_DIV");
            return e ? std::max(1, std::atoi(e)) : 0;
        }();
        dm.set_draft_grid(env ? env : (gamma <= 2 ? 2 : 1));
    }
    bool colocated_ = false;
    ~DoubleEngine() {
        dm.set_smem_budget(kFwdSmemBudget);
        tm.set_smem_budget(kFwdSmemBudget);
        dm.set_draft_grid(1);
    }
    bool split() const { return S.dmain != S.main; }

    // DBL_ROUND_TIMELINE_FILE=path (+ DBL_ROUND_TIMELINE_N rounds, default 64): per round, the device
    // intervals of the verify forward and of every draft segment (CUDA events, one GPU: one clock) and
    // the host's finish_round time, appended as JSON lines — the PSD draft-while-verify overlap record
    struct Timeline {
        FILE* f = nullptr;
        long left = 0, round = 0;
        cudaEvent_t ev0 = nullptr, tf_acc = nullptr;
        std::vector<cudaEvent_t> ds, de;
        void init(int gamma) {
            for (int j = static_cast<int>(ds.size()); j < gamma; ++j) {
                cudaEvent_t a, b;
                CUDA_CHECK(cudaEventCreate(&a));
                CUDA_CHECK(cudaEventCreate(&b));
                ds.push_back(a);
                de.push_back(b);
            }
            if (!ev0) {
                CUDA_CHECK(cudaEventCreate(&ev0));
                CUDA_CHECK(cudaEventCreate(&tf_acc));
            }
        }
        ~Timeline() {
            if (f) std::fclose(f);
            for (auto e : ds) cudaEventDestroy(e);
            for (auto e : de) cudaEventDestroy(e);
            if (ev0) cudaEventDestroy(ev0);
            if (tf_acc) cudaEventDestroy(tf_acc);
        }
    } tl_;
    bool timeline_on(int gamma) {
        if (tl_.round == 0 && !tl_.f) {
            const char* path = std::getenv("DBL_ROUND_TIMELINE_FILE");
            if (path && *path && !split()) {
                tl_.f = std::fopen(path, "a");
                const char* n = std::getenv("DBL_ROUND_TIMELINE_N");
                tl_.left = n ? std::atol(n) : 64;
            }
        }
        if (!tl_.f || tl_.left <= 0) return false;
        tl_.init(gamma);
        return true;
    }
    // the draft side's datastore for sequence q (see DoubleSeq::dst); DBL_STORE_MIRROR=1 forces a replica
    // on the same device (tests the replication path on one GPU)
    void bind_store(DoubleSeq& q, DeviceStore* st) const {
        q.st = st;
        q.mirror.reset();
        q.dst = st;
        const char* fe = std::getenv("DBL_STORE_MIRROR");
        const bool force = fe && fe[0] == '1';
        if (split() || force) {
            CUDA_CHECK(cudaStreamSynchronize(S.main));
            q.mirror = st->clone_to(dm.device());
            q.dst = q.mirror.get();
            q.dst->stats(q.mirror_base, S.dmain);
        }
    }
    // finish_round's datastore appends, applied to both replicas in the same order
    void record(DoubleSeq& q, int layer, const std::vector<int32_t>& before, const int32_t* add, size_t na) const {
        record_run(*q.st, layer, before, add, na, S.main);
        if (q.dst != q.st) {
            DeviceGuard g(q.dst->device());
            record_run(*q.dst, layer, before, add, na, S.dmain);
        }
    }
    // the replica's lookups count in the datastore's stats (LookupStats, datastore.hpp:39-67)
    void unbind_store(DoubleSeq& q) const {
        if (!q.mirror) return;
        int64_t now[6], delta[6];
        q.mirror->stats(now, S.dmain);
        for (int i = 0; i < 6; ++i) delta[i] = now[i] - q.mirror_base[i];
        q.st->add_stats(delta, S.main);
        q.mirror.reset();
        q.dst = q.st;
    }

    // lanes (capacity `cap` tokens), round record and sampled-loop buffers of one sequence
    void init_seq(DoubleSeq& q, DeviceStore* st, int cap, const dbl_pipeline_options& o) const {
        q.st = st;
        q.dst = st;
        if (o.temperature != 0.0 && dm.device() != tm.device())
            throw_invalid("sampled decoding (temperature > 0) needs the draft and target on one device");
        q.dl = std::make_unique<Lane>(dm, cap);
        q.tl = std::make_unique<Lane>(tm, cap);
        q.dio = std::make_unique<LaneIO>(q.dl.get());
        q.tio = std::make_unique<LaneIO>(q.tl.get());
        q.rr_buf.alloc(1);
        q.rr = q.rr_buf.p;
        q.rr_dev = q.rr_buf.dev();
        q.smp.reset();
        if (o.temperature != 0.0) {
            if (dm.vocab() != tm.vocab()) throw_invalid("draft and target vocabularies differ");
            const int d = o.depth, gamma = o.gamma;
            q.smp = std::make_unique<Sampled>(o.temperature, o.rng_seed, tm.vocab(), d + 1, gamma * (d + 1),
                                              gamma * (d + 1) + d + 2);
        }
    }

    // one forward over the given lanes: the lane's own forward for a single lane, else batched when the
    // rows fit one forward (<= 256), else one forward per lane
    void forward_set(Model& m, std::vector<Lane*>& ls, const std::vector<int>& bounds, cudaStream_t s) {
        if (ls.size() == 1) {
            m.forward(*ls[0], bounds[0], s);
            return;
        }
        int total = 0;
        for (int v : bounds) total += v;
        if (total <= m.max_forward_tokens() && total <= 256) {
            m.forward_lanes(ls, total, s);
        } else {
            for (size_t i = 0; i < ls.size(); ++i) m.forward(*ls[i], bounds[i], s);
        }
    }
    void dists_set(Model& m, std::vector<Lane*>& ls, const std::vector<int>& bounds, const std::vector<int>& rows,
                   const std::vector<double*>& outs, cudaStream_t s) {
        int total = 0;
        for (int v : bounds) total += v;
        if (ls.size() == 1 || (total <= m.max_forward_tokens() && total <= 256)) {
            m.dists_lanes(ls, total, rows, outs, s);
        } else {
            for (size_t i = 0; i < ls.size(); ++i) m.dists(*ls[i], bounds[i], rows[i], outs[i], s);
        }
    }

    // run_round (pipeline.cpp:223-262) for every sequence in `act`: each gets one Trace appended to
    // q.res.traces and its PipelineState advanced; lanes are left holding committed ⊕ speculative.
    void round(const std::vector<DoubleSeq*>& act, const dbl_pipeline_options& o) {
        NvtxRange nv_round("dbl.round");
        const int d = o.depth, gamma = o.gamma;
        const int c_max = o.draft_retrieval ? d : 0, tc_max = o.target_retrieval ? d : 0;
        for (DoubleSeq* qp : act) {
            DoubleSeq& q = *qp;
            // check_state, pipeline.cpp:208-219
            if (q.mode == 0 && !q.spec.empty()) throw_logic("pre-verify mode with a speculative tail");
            if (q.mode == 1 && q.prev_tokens != static_cast<int>(q.spec.size()))
                throw_logic("prev_tokens out of sync with speculative tail");
            q.nc = static_cast<int>(q.committed.size());
            q.ns = static_cast<int>(q.spec.size());
            q.L = q.nc + q.ns;
            q.rr->draft_L0 = q.L;
            q.rr->draft_L = q.L;
            q.rr->n_segs = 0;
            q.rr->draft_error = q.rr->target_error = 0;
            if (q.smp) launch_derive_rngs(q.smp->rng.p, q.smp->seed, static_cast<uint64_t>(q.round), S.main);
        }
        const bool tlon = timeline_on(gamma);
        const auto h0 = std::chrono::steady_clock::now();
        if (tlon) CUDA_CHECK(cudaEventRecord(tl_.ev0, S.main));
        S.fork();
        // ---- draft worker: iterative_draft over committed ⊕ spec (pipeline.cpp:39-46)
        std::vector<Lane*> dls, tls;
        std::vector<int> bounds;
        DeviceGuard gd(dm.device());
        auto nv_draft = std::make_unique<NvtxRange>("dbl.draft");
        for (int j = 0; j < gamma; ++j) {
            if (tlon) CUDA_CHECK(cudaEventRecord(tl_.ds[j], S.draft));
            dls.clear();
            bounds.clear();
            for (DoubleSeq* qp : act) {
                DoubleSeq& q = *qp;
                const int first = j == 0 ? split_long_forward(*q.dl, q.L, q.L - 1, c_max, q.smp != nullptr, S.draft) : 0;
                if (o.draft_retrieval) q.dst->lookup_lane(q.dl->buf.p, q.dl->state, d, S.draft);
                dls.push_back(q.dl.get());
                bounds.push_back(j == 0 ? q.L + c_max - first : 1 + c_max);
            }
            if (act[0]->smp) {
                std::vector<int> rows;
                std::vector<double*> outs;
                for (DoubleSeq* qp : act) {
                    rows.push_back(c_max + 1);
                    outs.push_back(qp->smp->ddist.p);
                }
                dists_set(dm, dls, bounds, rows, outs, S.draft);
                for (DoubleSeq* qp : act) {
                    DoubleSeq& q = *qp;
                    Sampled& sm = *q.smp;
                    launch_draft_accept_sampled(*q.dl, q.rr_dev, j, q.L, sm.ddist.p, sm.chain[sm.cur].p, sm.chain_rows,
                                                sm.rng.p, sm.T, sm.dscratch.p, S.draft);
                }
            } else {
                forward_set(dm, dls, bounds, S.draft);
                for (DoubleSeq* qp : act) launch_draft_accept(*qp->dl, qp->rr_dev, j, S.draft);
            }
            if (tlon) CUDA_CHECK(cudaEventRecord(tl_.de[j], S.draft));
        }
        nv_draft.reset();
        // ---- target worker: lookup + one batched verify forward (pipeline.cpp:48-70)
        DeviceGuard gt(tm.device());
        auto nv_target = std::make_unique<NvtxRange>("dbl.target");
        bounds.clear();
        for (DoubleSeq* qp : act) {
            DoubleSeq& q = *qp;
            const int first = split_long_forward(*q.tl, q.L, q.nc - 1, tc_max, q.smp != nullptr, S.target);
            if (o.target_retrieval) q.st->lookup_lane(q.tl->buf.p, q.tl->state, d, S.target);
            tls.push_back(q.tl.get());
            bounds.push_back(q.L + tc_max - first);
        }
        CUDA_CHECK(cudaEventRecord(S.tf0, S.target));
        if (act[0]->smp) {
            // verify forward + finish_round's verification (rng_v) + the target's own acceptance (rng_t)
            std::vector<int> rows;
            std::vector<double*> outs;
            for (DoubleSeq* qp : act) {
                rows.push_back(qp->ns + tc_max + 1);
                outs.push_back(qp->smp->tdist.p);
            }
            dists_set(tm, tls, bounds, rows, outs, S.target);
            CUDA_CHECK(cudaEventRecord(S.tf1, S.target));
            for (DoubleSeq* qp : act) {
                DoubleSeq& q = *qp;
                Sampled& sm = *q.smp;
                launch_target_accept_sampled(*q.tl, q.nc, q.rr_dev, sm.tdist.p, sm.spec_probs, sm.rng.p + 1,
                                             sm.rng.p + 2, sm.T, false, sm.tscratch.p, S.target);
            }
        } else {
            forward_set(tm, tls, bounds, S.target);
            CUDA_CHECK(cudaEventRecord(S.tf1, S.target));
            for (DoubleSeq* qp : act) launch_target_accept(*qp->tl, qp->nc, qp->rr_dev, S.target);
        }
        if (tlon) CUDA_CHECK(cudaEventRecord(tl_.tf_acc, S.target));
        nv_target.reset();
        {
            NvtxRange nv_wait("dbl.wait");
            CUDA_CHECK(cudaStreamSynchronize(S.draft));
            CUDA_CHECK(cudaStreamSynchronize(S.target));
        }
        const auto h1 = std::chrono::steady_clock::now();
        {
            float ms = 0.f;
            CUDA_CHECK(cudaEventElapsedTime(&ms, S.tf0, S.tf1));
            tfwd_ms += ms;
            ++tfwd_n;
        }
        {
            NvtxRange nv_fin("dbl.finish_round");
            for (DoubleSeq* qp : act) finish(*qp, o);
        }
        if (tlon) {
            const auto h2 = std::chrono::steady_clock::now();
            auto us = [&](cudaEvent_t e) {
                float ms = 0.f;
                CUDA_CHECK(cudaEventElapsedTime(&ms, tl_.ev0, e));
                return 1e3 * ms;
            };
            std::fprintf(tl_.f, "{\"round\":%ld,\"gamma\":%d,\"target_fwd\":[%.1f,%.1f],\"target_end\":%.1f,\"draft\":[",
                         tl_.round, gamma, us(S.tf0), us(S.tf1), us(tl_.tf_acc));
            for (int j = 0; j < gamma; ++j)
                std::fprintf(tl_.f, "%s[%.1f,%.1f]", j ? "," : "", us(tl_.ds[j]), us(tl_.de[j]));
            std::fprintf(tl_.f, "],\"host_wait_us\":%.1f,\"host_finish_us\":%.1f,\"target_rows\":%d}\n",
                         std::chrono::duration<double, std::micro>(h1 - h0).count(),
                         std::chrono::duration<double, std::micro>(h2 - h1).count(),
                         act[0]->L + act[0]->rr->ext_c - (act[0]->nc - 1));
            ++tl_.round;
            if (--tl_.left == 0) {
                std::fclose(tl_.f);
                tl_.f = nullptr;
            }
        }
    }

    // finish_round (pipeline.cpp:91-206) + rollback(state, |committed|) (pipeline.cpp:15-30) + the KV
    // commit of both lanes (kv_len := LCP of what the device processed and committed' ⊕ spec')
    void finish(DoubleSeq& q, const dbl_pipeline_options& o) {
        const int gamma = o.gamma;
        RoundResult* rr = q.rr;
        Lane& dl = *q.dl;
        Lane& tl = *q.tl;
        Sampled* smp = q.smp.get();
        const int L = q.L, nc = q.nc, ns = q.ns;
        if ((rr->draft_error || rr->target_error) && std::getenv("DBL_DEBUG_ROUND"))
            std::fprintf(stderr, "dbl round %ld: draft_error %d target_error %d L %d nc %d ns %d n_segs %d draft_L %d ext_c %d\n",
                         q.round, rr->draft_error, rr->target_error, L, nc, ns, rr->n_segs, rr->draft_L, rr->ext_c);
        check_round_errors(rr);
        const int c_t = rr->ext_c;
        q.trows += L + c_t - (nc - 1);

        const int n_chain = rr->draft_L - rr->draft_L0;
        const int32_t* chain = rr->draft_tokens;
        const int ne = rr->ext_matched + 1;
        const int32_t* ext = rr->ext_emitted;
        Trace tr;
        tr.round = q.round;
        tr.mode = q.mode ? "post_verify" : "pre_verify";
        tr.pending = ns;
        tr.draft_len = n_chain;
        if (o.draft_retrieval)
            for (int j = 0; j < rr->n_segs; ++j) tr.draft_matched.push_back(rr->segs[j].matched);
        tr.target_matched = o.target_retrieval ? rr->ext_matched : -1;
        tr.target_source = source_name(rr->ext_source);

        const std::vector<int32_t> committed_before = q.committed;
        std::vector<int32_t> add, new_spec;
        const std::vector<int32_t>& spec = q.spec;
        if (smp) smp->spec_probs = nullptr;
        if (rr->tgt_rej >= 0) {
            const int k = rr->tgt_rej;
            tr.accepted_pending = k;
            tr.pending_reject = tr.rejected = true;
            tr.kind = "pending_reject";
            add.assign(spec.begin(), spec.begin() + k);
            add.push_back(rr->tgt_correction);
            std::vector<int32_t> pre_k = committed_before;
            pre_k.insert(pre_k.end(), spec.begin(), spec.begin() + k);
            record(q, 2, pre_k, spec.data() + k, spec.size() - k);
            std::vector<int32_t> pre_d = committed_before;
            pre_d.insert(pre_d.end(), spec.begin(), spec.end());
            record(q, 2, pre_d, chain, n_chain);
        } else {
            tr.accepted_pending = ns;
            add = spec;
            add.insert(add.end(), ext, ext + ne);
            const int cmp = std::min(n_chain, ne);
            int j = 0;
            while (j < cmp && chain[j] == ext[j]) ++j;
            if (j == ne && n_chain > ne) {
                tr.kind = "extend_keep_draft";
                new_spec.assign(chain + ne, chain + n_chain);
                if (smp) {  // new_spec_probs = chain.probs[ne:] (pipeline.cpp:168-169)
                    smp->spec_probs = smp->chain[smp->cur].p + static_cast<size_t>(ne) * smp->V;
                    smp->cur ^= 1;
                }
            } else if (j == cmp) {
                tr.kind = "extend_draft_subsumed";
            } else {
                tr.kind = "extend_drop_draft";
                tr.rejected = true;
                std::vector<int32_t> pre_j = committed_before;
                pre_j.insert(pre_j.end(), spec.begin(), spec.end());
                pre_j.insert(pre_j.end(), chain, chain + j);
                record(q, 2, pre_j, chain + j, n_chain - j);
            }
        }
        tr.committed_count = static_cast<int>(add.size());
        record(q, 1, committed_before, add.data(), add.size());
        q.committed.insert(q.committed.end(), add.begin(), add.end());
        // rollback(state, |committed|) (pipeline.cpp:15-30)
        if (static_cast<long>(q.committed.size()) < q.last_committed_len)
            throw_logic("rollback: keep_len below committed boundary");
        q.spec = std::move(new_spec);
        q.mode = q.spec.empty() ? 0 : 1;
        q.prev_tokens = q.spec.empty() ? gamma : static_cast<int>(q.spec.size());
        q.last_committed_len = static_cast<long>(q.committed.size());
        ++q.round;
        const double draft_time = gamma * (o.t_draft + (o.draft_retrieval ? o.t_lookup : 0.0));
        const double target_time = o.t_target + (o.target_retrieval ? o.t_lookup : 0.0);
        tr.clock_delta = std::max(draft_time, target_time) + o.t_sync;
        q.res.traces.push_back(std::move(tr));
        {  // decision log (see RunOutput::log)
            auto& lg = q.res.log;
            lg.push_back(rr->n_segs);
            int at = 0;
            for (int j = 0; j < rr->n_segs; ++j) {
                lg.push_back(rr->segs[j].matched);
                lg.insert(lg.end(), chain + at, chain + at + rr->segs[j].n_emit);
                at += rr->segs[j].n_emit;
            }
            lg.push_back(ns);
            lg.push_back(rr->tgt_rej);
            lg.push_back(rr->tgt_correction);
            lg.push_back(rr->ext_matched);
            lg.insert(lg.end(), ext, ext + ne);
        }

        // ---- lane cursors for the next round (KV commit by length)
        // the draft lane holds committed_before ⊕ spec ⊕ chain; KV valid below its last token
        dl.mirror.resize(L);
        dl.mirror.insert(dl.mirror.end(), chain, chain + n_chain);
        dl.kv_len = L + n_chain - 1;  // sync() takes the LCP with committed' ⊕ spec'
        tl.mirror.resize(L);
        tl.mirror.insert(tl.mirror.end(), rr->ext_cands, rr->ext_cands + c_t);
        tl.kv_len = L + c_t;
        sync(q);
    }

    // make both lanes hold committed ⊕ speculative with KV valid for the longest common prefix of what
    // they processed (the "rollback-free" commit: nothing moves, only kv_len)
    void sync(DoubleSeq& q) {
        std::vector<int32_t> X = q.committed;
        X.insert(X.end(), q.spec.begin(), q.spec.end());
        const int n = static_cast<int>(X.size()), nc = static_cast<int>(q.committed.size());
        Lane& dl = *q.dl;
        Lane& tl = *q.tl;
        {
            DeviceGuard g(dm.device());
            dl.kv_len = std::min(dl.kv_len, q.dio->sync_tokens(X, S.dmain));
            dl.set_state(n, 0, dl.kv_len, n - 1, S.dmain);
        }
        tl.kv_len = std::min(tl.kv_len, q.tio->sync_tokens(X, S.main));
        tl.set_state(n, 0, tl.kv_len, nc - 1, S.main);
    }
};
}  // namespace

// run (pipeline.cpp:264-323) for one or several independent sequences.  With B > 1 every draft
// segment and every verify step is ONE forward over all active sequences (Model::forward_lanes), and
// the per-sequence acceptance, finish_round and datastore updates are unchanged — so each sequence's
// output, traces and metrics equal its own single-sequence run.  B = 1 issues exactly the device
// work of the single-sequence loop.
std::vector<RunOutput> run_double_multi(Model& dm, Model& tm, const std::vector<DeviceStore*>& stores,
                                        const std::vector<std::vector<int32_t>>& prompts, int max_new,
                                        const dbl_pipeline_options& o) {
    const int B = static_cast<int>(prompts.size());
    if (B < 1 || B > kMaxBatchSeqs || static_cast<int>(stores.size()) != B)
        throw_invalid("run: 1.." + std::to_string(kMaxBatchSeqs) + " sequences, one datastore each");
    if (max_new < 1) throw_invalid("max_new_tokens must be >= 1");
    for (const auto& p : prompts)
        if (p.empty()) throw_invalid("prompt must be nonempty");
    validate_opts(o);
    for (DeviceStore* st : stores)
        if (tm.device() != st->device()) throw_invalid("the datastore must live on the target's device");
    for (int i = 0; i < B; ++i)
        for (int k = i + 1; k < B; ++k)
            if (stores[i] == stores[k]) throw_invalid("batched run: every sequence needs its own datastore");
    DeviceGuard g(stores[0]->device());
    const int d = o.depth, gamma = o.gamma;
    size_t longest = 0;
    for (const auto& p : prompts) longest = std::max(longest, p.size());
    const int cap = static_cast<int>(longest) + max_new + 3 * gamma * (d + 1) + 3 * d + 64;
    DoubleEngine E(dm, tm);
    E.configure_draft(gamma);
    Streams& S = E.S;

    std::vector<DoubleSeq> seqs(B);
    for (int b = 0; b < B; ++b) {
        DoubleSeq& q = seqs[b];
        E.init_seq(q, stores[b], cap, o);
        E.bind_store(q, stores[b]);
        device_counts(*q.st, S.main, &q.base_lookups, &q.base_hits);
        q.n_prompt = static_cast<int>(prompts[b].size());
        q.committed = prompts[b];
        q.prev_tokens = gamma;
        q.last_committed_len = q.n_prompt;
        q.scanned = q.n_prompt;
        q.st->record(1, prompts[b].data(), q.n_prompt, S.main);  // store.record_accepted(prompt), pipeline.cpp:282
        if (q.dst != q.st) q.dst->record(1, prompts[b].data(), q.n_prompt, S.dmain);
        // lanes hold the prompt; transformers prefill KV for positions [0, P-1)
        {
            DeviceGuard gd(dm.device());
            q.dio->sync_tokens(q.committed, S.dmain);
        }
        q.tio->sync_tokens(q.committed, S.main);
    }
    Timer pre;
    CUDA_CHECK(cudaEventRecord(pre.a, S.main));
    S.fork();
    for (DoubleSeq& q : seqs) {
        {
            DeviceGuard gd(dm.device());
            catch_up(*q.dl, q.n_prompt - 1, S.draft);
        }
        catch_up(*q.tl, q.n_prompt - 1, S.target);
    }
    S.join_draft_into_main();
    if (E.split()) CUDA_CHECK(cudaStreamWaitEvent(S.dmain, S.dready, 0));  // the draft lane's cursor after its prefill
    CUDA_CHECK(cudaEventRecord(S.ready, S.target));
    CUDA_CHECK(cudaStreamWaitEvent(S.main, S.ready, 0));
    CUDA_CHECK(cudaEventRecord(pre.b, S.main));
    for (DoubleSeq& q : seqs) {
        {
            DeviceGuard gd(dm.device());
            q.dl->set_state(q.n_prompt, 0, q.dl->kv_len, q.n_prompt - 1, S.dmain);
        }
        q.tl->set_state(q.n_prompt, 0, q.tl->kv_len, q.n_prompt - 1, S.main);
    }

    Timer loop;
    CUDA_CHECK(cudaEventRecord(loop.a, S.main));
    const long long launches0 = launch_counter();
    const int32_t eos = tm.vocab() - 1;
    std::vector<DoubleSeq*> act;
    for (;;) {
        act.clear();
        for (DoubleSeq& q : seqs)
            if (!q.done) act.push_back(&q);
        if (act.empty()) break;
        E.round(act, o);
        for (DoubleSeq* qp : act) {  // EOS / budget (pipeline.cpp:290-306)
            DoubleSeq& q = *qp;
            for (; q.scanned < q.committed.size(); ++q.scanned) {
                if (q.committed[q.scanned] == eos) {
                    q.committed.resize(q.scanned + 1);
                    q.done = true;
                    break;
                }
            }
            if (q.committed.size() - static_cast<size_t>(q.n_prompt) >= static_cast<size_t>(max_new)) q.done = true;
            if (q.round > 1000000) throw_runtime("round limit exceeded; pipeline stalled");
        }
    }
    CUDA_CHECK(cudaEventRecord(loop.b, S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.dmain));

    std::vector<RunOutput> out;
    for (DoubleSeq& q : seqs) {
        E.unbind_store(q);
        RunOutput& res = q.res;
        finish_output(q.committed, q.n_prompt, max_new, res);
        compute_metrics(res.traces, o.t_target, &res.metrics);
        long lk, hits;
        device_counts(*q.st, S.main, &lk, &hits);
        res.metrics.lookups = lk - q.base_lookups;
        res.metrics.hit_rate = res.metrics.lookups == 0
                                   ? 0.0
                                   : static_cast<double>(hits - q.base_hits) / static_cast<double>(res.metrics.lookups);
        res.metrics.device_ms = loop.ms();
        res.metrics.kernel_launches = launch_counter() - launches0;
        res.metrics.prefill_ms = pre.ms();
        res.metrics.target_fwd_ms = E.tfwd_ms;
        res.metrics.target_fwd_count = E.tfwd_n;
        res.metrics.target_rows = q.trows;
        q.st->flush_session(S.main);  // pipeline.cpp:321
        out.push_back(std::move(res));
    }
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    return out;
}

RunOutput run_double(Model& dm, Model& tm, DeviceStore& st, const int32_t* prompt, int n_prompt, int max_new,
                     const dbl_pipeline_options& o) {
    if (max_new < 1) throw_invalid("max_new_tokens must be >= 1");
    if (n_prompt <= 0) throw_invalid("prompt must be nonempty");
    std::vector<RunOutput> r = run_double_multi(dm, tm, {&st}, {std::vector<int32_t>(prompt, prompt + n_prompt)},
                                                max_new, o);
    return std::move(r[0]);
}

// ------------------------------------------------------------------------ run_round session
// A PipelineState driven one round at a time (run_round, pipeline.cpp:223-262).  The session keeps
// the two lanes (token buffers + KV) between calls; each call re-synchronises them with the state it
// is given by longest common prefix, so any state — a fresh one, a rolled-back one, a copy — runs
// exactly as the reference would, and an unchanged state pays nothing.
struct RoundSession::Impl {
    DoubleEngine E;
    std::unique_ptr<DoubleSeq> q;
    int cap = 0, gamma = 0, depth = 0;
    double temperature = 0.0;
    uint64_t seed = 0;
    bool dev_spec_valid = false;  // the sampled loop's spec_probs rows on the device belong to last_spec
    std::vector<int32_t> last_spec;
    const double* spec_dev = nullptr;
    Impl(Model& d, Model& t) : E(d, t) {}
};

RoundSession::RoundSession(Model& dm, Model& tm) {
    if (dm.device() != tm.device()) throw_invalid("draft and target must live on the same device");
    DeviceGuard g(tm.device());
    impl_ = std::make_unique<Impl>(dm, tm);
}
RoundSession::~RoundSession() = default;

Trace RoundSession::run_round(HostPipelineState& st, DeviceStore& store, const dbl_pipeline_options& o,
                              std::vector<double>* spec_probs_out) {
    Impl& I = *impl_;
    validate_opts(o);
    // check_state (pipeline.cpp:208-219)
    if (st.mode == 0 && !st.speculative.empty()) throw_logic("pre-verify mode with a speculative tail");
    if (st.mode == 1 && st.prev_tokens != static_cast<int>(st.speculative.size()))
        throw_logic("prev_tokens out of sync with speculative tail");
    if (static_cast<long>(st.speculative.size()) != st.n_spec_probs)
        throw_logic("speculative tokens and probs out of sync");
    if (st.committed.empty()) throw_invalid("forward_batch: empty context");  // model.cpp:41
    if (store.device() != I.E.tm.device() || I.E.dm.device() != I.E.tm.device())
        throw_invalid("run_round: draft, target and datastore must live on the same device");
    DeviceGuard g(store.device());
    const int n = static_cast<int>(st.committed.size() + st.speculative.size());
    const int need = n + 3 * o.gamma * (o.depth + 1) + 3 * o.depth + 64;
    const bool sampled = o.temperature != 0.0;
    if (!I.q || need > I.cap || o.gamma != I.gamma || o.depth != I.depth || o.temperature != I.temperature ||
        o.rng_seed != I.seed) {
        const int cap = std::max(need, I.cap) + 256;
        I.q.reset();  // its lanes' caches go back to the models first
        I.q = std::make_unique<DoubleSeq>();
        I.E.configure_draft(o.gamma);
        I.E.init_seq(*I.q, &store, cap, o);
        I.cap = cap;
        I.gamma = o.gamma;
        I.depth = o.depth;
        I.temperature = o.temperature;
        I.seed = o.rng_seed;
        I.dev_spec_valid = false;
    }
    DoubleSeq& q = *I.q;
    q.st = &store;
    q.dst = &store;  // one device (checked above): the draft side reads the same datastore
    // the caller may have changed the datastore since the last round (API calls run on the legacy
    // stream; the session's streams are non-blocking): order this round after that work
    CUDA_CHECK(cudaEventRecord(I.E.S.ready, 0));
    CUDA_CHECK(cudaStreamWaitEvent(I.E.S.main, I.E.S.ready, 0));
    q.committed = st.committed;
    q.spec = st.speculative;
    q.mode = st.mode;
    q.prev_tokens = st.prev_tokens;
    q.round = st.round;
    q.last_committed_len = st.last_committed_len;
    q.res.traces.clear();
    q.res.log.clear();
    if (sampled) {
        Sampled& sm = *q.smp;
        sm.spec_probs = nullptr;
        if (!q.spec.empty()) {
            if (st.spec_probs_in) {  // the caller's rows -> the chain buffer the next draft does not write
                const size_t rows = q.spec.size();
                if (rows > static_cast<size_t>(sm.chain_rows)) throw_invalid("speculative tail longer than gamma * (depth + 1)");
                double* dst = sm.chain[sm.cur ^ 1].p;
                CUDA_CHECK(cudaMemcpyAsync(dst, st.spec_probs_in, rows * sm.V * sizeof(double), cudaMemcpyHostToDevice,
                                           I.E.S.main));
                sm.spec_probs = dst;
            } else if (I.dev_spec_valid && I.last_spec == q.spec) {
                sm.spec_probs = I.spec_dev;
            } else {
                throw_invalid("run_round: spec_probs rows are required at temperature > 0");
            }
        }
    }
    I.E.sync(q);
    I.E.round({&q}, o);
    Trace tr = q.res.traces.back();
    st.committed = q.committed;
    st.speculative = q.spec;
    st.n_spec_probs = static_cast<long>(q.spec.size());
    st.mode = q.mode;
    st.prev_tokens = q.prev_tokens;
    st.round = q.round;
    st.last_committed_len = q.last_committed_len;
    st.clock += tr.clock_delta;  // state.clock.charge (pipeline.cpp:203)
    I.dev_spec_valid = sampled && !q.spec.empty();
    I.last_spec = q.spec;
    I.spec_dev = sampled ? q.smp->spec_probs : nullptr;
    if (spec_probs_out) {
        spec_probs_out->clear();
        if (I.dev_spec_valid) {
            spec_probs_out->resize(q.spec.size() * q.smp->V);
            CUDA_CHECK(cudaMemcpyAsync(spec_probs_out->data(), I.spec_dev, spec_probs_out->size() * sizeof(double),
                                       cudaMemcpyDeviceToHost, I.E.S.main));
        }
    }
    CUDA_CHECK(cudaStreamSynchronize(I.E.S.main));
    return tr;
}

// ----------------------------------------------------------------------------------- run (AR)
namespace {
__global__ void ar_append_kernel(const int32_t* __restrict__ argmax, int32_t* buf, LaneState* lane,
                                 int32_t* out_host, int i) {
    const int L = lane->L;
    const int tok = argmax[L - 1];
    buf[L] = tok;
    out_host[i] = tok;
    if (tok < 0) lane->error = 1;
    lane->L = L + 1;
    lane->c = 0;
    lane->kv_len = L;
    lane->row0 = L;
}
}  // namespace

RunOutput run_ar(Model& tm, const int32_t* prompt, int n_prompt, int max_new, double t_target,
                 double temperature, uint64_t seed) {
    // run_vanilla_ar, harness.cpp:233-258.  The device runs ahead in blocks of kBlock tokens between
    // EOS checks; tokens past an EOS are discarded exactly as the reference never produces them (at
    // temperature > 0 the extra draws come after every kept token's, so kept tokens are unaffected).
    if (n_prompt <= 0) throw_invalid("prompt must be nonempty");
    if (max_new < 0) throw_invalid("max_new_tokens must be >= 0");
    if (!(temperature >= 0.0)) throw_invalid("temperature must be >= 0");
    DeviceGuard g(tm.device());
    constexpr int kBlock = 16;
    const int cap = n_prompt + max_new + kBlock + 8;
    Streams S;
    Lane tl(tm, cap);
    LaneIO tio(&tl);
    PinBuf<int32_t> outp(std::max(max_new + kBlock, 1));
    int32_t* out_dev = outp.dev();
    std::vector<int32_t> ctx(prompt, prompt + n_prompt);
    tio.sync_tokens(ctx, S.main);
    Timer pre, loop;
    CUDA_CHECK(cudaEventRecord(pre.a, S.main));
    catch_up(tl, n_prompt - 1, S.main);
    CUDA_CHECK(cudaEventRecord(pre.b, S.main));
    tl.set_state(n_prompt, 0, tl.kv_len, n_prompt - 1, S.main);
    std::unique_ptr<Sampled> smp;
    if (temperature != 0.0) {
        smp = std::make_unique<Sampled>(temperature, seed, tm.vocab(), 0, 0, 1);
        launch_seed_rng(smp->rng.p, splitmix64(seed ^ 0x6172000000000000ULL), S.main);  // harness.cpp:235
    }
    CUDA_CHECK(cudaEventRecord(loop.a, S.main));
    const long long launches0 = launch_counter();
    RunOutput res;
    const int32_t eos = tm.vocab() - 1;
    int produced = 0;
    bool done = max_new == 0;
    while (!done) {
        NvtxRange nv_blk("dbl.ar_block");
        const int n = std::min(kBlock, max_new - produced);
        for (int i = 0; i < n; ++i) {
            if (smp) {
                tm.dists(tl, 1, 1, smp->tdist.p, S.main);
                launch_ar_sample(tl, smp->tdist.p, smp->rng.p, smp->T, smp->tscratch.p, out_dev, produced + i,
                                 S.main);
            } else {
                tm.forward(tl, 1, S.main);
                ar_append_kernel<<<1, 1, 0, S.main>>>(tl.argmax.p, tl.buf.p, tl.state, out_dev, produced + i);
                CUDA_LAUNCH_CHECK();
            }
        }
        CUDA_CHECK(cudaStreamSynchronize(S.main));
        for (int i = 0; i < n; ++i) {
            const int32_t tok = outp.p[produced + i];
            if (tok < 0) raise_sample_error(smp ? -tok - 1 : kSampDegenerate);
            res.output.push_back(tok);
            Trace t;
            t.round = produced + i;
            t.mode = "ar";
            t.committed_count = 1;
            t.kind = "ar_step";
            t.clock_delta = t_target;
            res.traces.push_back(std::move(t));
            if (tok == eos) { done = true; break; }
        }
        produced += n;
        if (produced >= max_new) done = true;
    }
    CUDA_CHECK(cudaEventRecord(loop.b, S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    compute_metrics(res.traces, t_target, &res.metrics);
    res.metrics.clock = static_cast<double>(res.metrics.tokens) * t_target;  // harness.cpp:254-256
    res.metrics.speedup = 1.0;
    res.metrics.device_ms = loop.ms();
    res.metrics.kernel_launches = launch_counter() - launches0;
    res.metrics.prefill_ms = pre.ms();
    res.metrics.target_fwd_count = produced;
    res.metrics.target_rows = produced;
    return res;
}

// ------------------------------------------------------------------------- run (batched AR)
namespace {
struct AppendBatch {
    const int32_t* argmax[kMaxBatchSeqs];
    int32_t* buf[kMaxBatchSeqs];
    LaneState* st[kMaxBatchSeqs];
    int n, stride;
};
__global__ void ar_append_batch_kernel(AppendBatch ab, int32_t* out_host, int i) {
    const int b = threadIdx.x;
    if (b >= ab.n) return;
    LaneState* lane = ab.st[b];
    const int L = lane->L;
    const int tok = ab.argmax[b][L - 1];
    ab.buf[b][L] = tok;
    out_host[b * ab.stride + i] = tok;
    if (tok < 0) lane->error = 1;
    lane->L = L + 1;
    lane->c = 0;
    lane->kv_len = L;
    lane->row0 = L;
}
}  // namespace

std::vector<RunOutput> run_ar_batch(Model& tm, const std::vector<std::vector<int32_t>>& prompts, int max_new,
                                    double t_target, double* device_ms, long long* launches) {
    // run_vanilla_ar (harness.cpp:233-258) for B independent sequences in lockstep: every step is ONE
    // forward over the B lanes (one row each) — the weight stream is shared, so B sequences cost about
    // one.  Each output equals that sequence's own run_vanilla_ar (greedy, bitwise: a row's arithmetic
    // never depends on the other rows).
    const int B = static_cast<int>(prompts.size());
    if (B < 1 || B > kMaxBatchSeqs) throw_invalid("run_ar_batch: 1.." + std::to_string(kMaxBatchSeqs) + " sequences");
    if (max_new < 0) throw_invalid("max_new_tokens must be >= 0");
    size_t longest = 0;
    for (const auto& p : prompts) {
        if (p.empty()) throw_invalid("prompt must be nonempty");
        longest = std::max(longest, p.size());
    }
    DeviceGuard g(tm.device());
    constexpr int kBlock = 16;
    const int cap = static_cast<int>(longest) + max_new + kBlock + 8;
    Streams S;
    std::vector<std::unique_ptr<Lane>> lanes;
    std::vector<std::unique_ptr<LaneIO>> ios;
    std::vector<Lane*> lp;
    AppendBatch ab{};
    ab.n = B;
    const int stride = std::max(max_new + kBlock, 1);
    ab.stride = stride;
    for (int b = 0; b < B; ++b) {
        lanes.push_back(std::make_unique<Lane>(tm, cap));
        Lane& l = *lanes.back();
        ios.push_back(std::make_unique<LaneIO>(&l));
        ios.back()->sync_tokens(prompts[b], S.main);
        catch_up(l, static_cast<int>(prompts[b].size()) - 1, S.main);
        const int n = static_cast<int>(prompts[b].size());
        l.set_state(n, 0, l.kv_len, n - 1, S.main);
        lp.push_back(&l);
        ab.argmax[b] = l.argmax.p;
        ab.buf[b] = l.buf.p;
        ab.st[b] = l.state;
    }
    PinBuf<int32_t> outp(static_cast<size_t>(B) * stride);
    int32_t* out_dev = outp.dev();
    Timer loop;
    CUDA_CHECK(cudaEventRecord(loop.a, S.main));
    const long long launches0 = launch_counter();
    std::vector<RunOutput> res(B);
    std::vector<char> done(B, max_new == 0 ? 1 : 0);
    const int32_t eos = tm.vocab() - 1;
    int produced = 0;
    while (produced < max_new && std::count(done.begin(), done.end(), 0) > 0) {
        const int n = std::min(kBlock, max_new - produced);
        for (int i = 0; i < n; ++i) {
            tm.forward_lanes(lp, B, S.main);
            ar_append_batch_kernel<<<1, 32, 0, S.main>>>(ab, out_dev, produced + i);
            CUDA_LAUNCH_CHECK();
        }
        CUDA_CHECK(cudaStreamSynchronize(S.main));
        for (int b = 0; b < B; ++b) {
            for (int i = 0; i < n && !done[b]; ++i) {
                const int32_t tok = outp.p[static_cast<size_t>(b) * stride + produced + i];
                if (tok < 0) throw_runtime("degenerate distribution");
                res[b].output.push_back(tok);
                Trace t;
                t.round = produced + i;
                t.mode = "ar";
                t.committed_count = 1;
                t.kind = "ar_step";
                t.clock_delta = t_target;
                res[b].traces.push_back(std::move(t));
                if (tok == eos) done[b] = 1;
            }
        }
        produced += n;
    }
    CUDA_CHECK(cudaEventRecord(loop.b, S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    for (auto& r : res) {
        compute_metrics(r.traces, t_target, &r.metrics);
        r.metrics.clock = static_cast<double>(r.metrics.tokens) * t_target;
        r.metrics.speedup = 1.0;
    }
    if (device_ms) *device_ms = loop.ms();
    if (launches) *launches = launch_counter() - launches0;
    return res;
}

// ---------------------------------------------------------------------------- run (serial SD)
RunOutput run_serial_sd(Model& dm, Model& tm, DeviceStore& st, const int32_t* prompt, int n_prompt,
                        int max_new, const dbl_pipeline_options& o, bool use_retrieval) {
    // run_serial_sd, harness.cpp:264-369 (greedy): draft chain over committed, one target forward
    // over committed ⊕ chain, accept prefix + correction or all + bonus token.
    if (n_prompt <= 0) throw_invalid("prompt must be nonempty");
    validate_opts(o);
    DeviceGuard g(st.device());
    const int d = o.depth, gamma = o.gamma;
    const int cap = n_prompt + max_new + 3 * gamma * (d + 1) + 3 * d + 64;
    Streams S;
    Lane dl(dm, cap), tl(tm, cap);
    LaneIO dio(&dl), tio(&tl);
    PinBuf<RoundResult> rr_buf(1);
    RoundResult* rr = rr_buf.p;
    RoundResult* rr_dev = rr_buf.dev();
    std::unique_ptr<Sampled> smp;
    if (o.temperature != 0.0) {
        if (dm.vocab() != tm.vocab()) throw_invalid("draft and target vocabularies differ");
        smp = std::make_unique<Sampled>(o.temperature, o.rng_seed, tm.vocab(), d + 1, gamma * (d + 1),
                                        gamma * (d + 1) + 1);
    }
    long base_lookups, base_hits;
    device_counts(st, S.main, &base_lookups, &base_hits);
    st.record(1, prompt, n_prompt, S.main);
    std::vector<int32_t> committed(prompt, prompt + n_prompt);
    dio.sync_tokens(committed, S.main);
    tio.sync_tokens(committed, S.main);
    catch_up(dl, n_prompt - 1, S.main);
    catch_up(tl, n_prompt - 1, S.main);
    RunOutput res;
    Timer loop;
    CUDA_CHECK(cudaEventRecord(loop.a, S.main));
    const long long launches0 = launch_counter();
    const int32_t eos = tm.vocab() - 1;
    long round = 0;
    size_t scanned = n_prompt;
    bool done = false;
    while (!done) {
        const int nc = static_cast<int>(committed.size());
        dl.set_state(nc, 0, dl.kv_len, nc - 1, S.main);
        rr->draft_L0 = rr->draft_L = nc;
        rr->n_segs = 0;
        rr->draft_error = rr->target_error = 0;
        // rng_d / rng_v = derive_rng(seed, round, 0 / 2) (harness.cpp:281-282)
        if (smp) launch_derive_rngs(smp->rng.p, smp->seed, static_cast<uint64_t>(round), S.main);
        for (int j = 0; j < gamma; ++j) {
            const int c_max = use_retrieval ? d : 0;
            const int first = j == 0 ? split_long_forward(dl, nc, nc - 1, c_max, smp != nullptr, S.main) : 0;
            if (use_retrieval) st.lookup_lane(dl.buf.p, dl.state, d, S.main);
            const int bound = j == 0 ? nc + c_max - first : 1 + c_max;
            if (smp) {
                dm.dists(dl, bound, c_max + 1, smp->ddist.p, S.main);
                launch_draft_accept_sampled(dl, rr_dev, j, nc, smp->ddist.p, smp->chain[0].p, smp->chain_rows,
                                            smp->rng.p, smp->T, smp->dscratch.p, S.main);
            } else {
                dm.forward(dl, bound, S.main);
                launch_draft_accept(dl, rr_dev, j, S.main);
            }
        }
        CUDA_CHECK(cudaStreamSynchronize(S.main));
        if (rr->draft_error) raise_sample_error(rr->draft_error);
        const int n_chain = rr->draft_L - rr->draft_L0;
        std::vector<int32_t> chain(rr->draft_tokens, rr->draft_tokens + n_chain);
        // target lane: chain as the "speculative" tail, no candidates
        std::vector<int32_t> X = committed;
        X.insert(X.end(), chain.begin(), chain.end());
        const int lcp = tio.sync_tokens(X, S.main);
        tl.kv_len = std::min(tl.kv_len, lcp);
        tl.set_state(nc + n_chain, 0, tl.kv_len, nc - 1, S.main);
        const int tbound = nc + n_chain - split_long_forward(tl, nc + n_chain, nc - 1, 0, smp != nullptr, S.main);
        if (smp) {
            tm.dists(tl, tbound, n_chain + 1, smp->tdist.p, S.main);
            launch_target_accept_sampled(tl, nc, rr_dev, smp->tdist.p, smp->chain[0].p, smp->rng.p + 1,
                                         smp->rng.p + 2, smp->T, true, smp->tscratch.p, S.main);
        } else {
            tm.forward(tl, tbound, S.main);
            launch_target_accept(tl, nc, rr_dev, S.main);
        }
        CUDA_CHECK(cudaStreamSynchronize(S.main));
        if (rr->target_error) raise_sample_error(rr->target_error);
        tl.kv_len = nc + n_chain;
        dl.mirror.resize(nc);
        dl.mirror.insert(dl.mirror.end(), chain.begin(), chain.end());
        dl.kv_len = nc + n_chain - 1;  // set by the last draft_accept on the device

        Trace t;
        t.round = round;
        t.mode = "serial";
        t.draft_len = n_chain;
        if (use_retrieval)
            for (int j = 0; j < rr->n_segs; ++j) t.draft_matched.push_back(rr->segs[j].matched);
        std::vector<int32_t> add;
        if (rr->tgt_rej >= 0) {
            const int k = rr->tgt_rej;
            t.accepted_pending = k;
            t.pending_reject = t.rejected = true;
            t.kind = "reject";
            add.assign(chain.begin(), chain.begin() + k);
            add.push_back(rr->tgt_correction);
            std::vector<int32_t> pre = committed;
            pre.insert(pre.end(), chain.begin(), chain.begin() + k);
            record_run(st, 2, pre, chain.data() + k, chain.size() - k, S.main);
        } else {
            t.accepted_pending = n_chain;
            t.kind = "all_accepted";
            add = chain;
            add.push_back(rr->ext_emitted[0]);  // sample(dists.back()), greedy
        }
        t.committed_count = static_cast<int>(add.size());
        t.clock_delta = gamma * (o.t_draft + (use_retrieval ? o.t_lookup : 0.0)) + o.t_target + o.t_sync;
        record_run(st, 1, committed, add.data(), add.size(), S.main);
        committed.insert(committed.end(), add.begin(), add.end());
        res.traces.push_back(std::move(t));
        ++round;
        // both lanes now must hold `committed`
        const int l1 = dio.sync_tokens(committed, S.main);
        dl.kv_len = std::min(dl.kv_len, l1);
        const int l2 = tio.sync_tokens(committed, S.main);
        tl.kv_len = std::min(tl.kv_len, l2);
        for (; scanned < committed.size(); ++scanned) {
            if (committed[scanned] == eos) {
                committed.resize(scanned + 1);
                done = true;
                break;
            }
        }
        if (committed.size() - static_cast<size_t>(n_prompt) >= static_cast<size_t>(max_new)) done = true;
        if (round > 1000000) throw_runtime("round limit exceeded; decoder stalled");
    }
    CUDA_CHECK(cudaEventRecord(loop.b, S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    finish_output(committed, n_prompt, max_new, res);
    compute_metrics(res.traces, o.t_target, &res.metrics);
    long lk, hits;
    device_counts(st, S.main, &lk, &hits);
    res.metrics.lookups = lk - base_lookups;
    res.metrics.hit_rate = res.metrics.lookups == 0
                               ? 0.0
                               : static_cast<double>(hits - base_hits) / static_cast<double>(res.metrics.lookups);
    res.metrics.device_ms = loop.ms();
    res.metrics.kernel_launches = launch_counter() - launches0;
    return res;
}

// ------------------------------------------------------------------------ stateless forward
namespace {
__global__ void gather_rows_kernel(const int32_t* argmax, int from, int n, int32_t* out) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = argmax[from + i];
}
}  // namespace

void forward_stateless(Model& m, const int32_t* ctx, int L, const int32_t* cands, int c,
                       int32_t* out_argmax, float* out_logits, double* out_dists, DevBuf<double>* keep_dists) {
    if (L <= 0) throw_invalid("forward_batch: empty context");  // model.cpp:41
    if (c < 0) throw_invalid("negative candidate count");
    DeviceGuard g(m.device());
    Streams S;
    Lane lane(m, L + c + 16);
    LaneIO io(&lane);
    std::vector<int32_t> X(ctx, ctx + L);
    X.insert(X.end(), cands, cands + c);
    io.sync_tokens(X, S.main);
    catch_up(lane, L - 1, S.main);
    DevBuf<float> lg;
    DevBuf<double> dd;
    if (keep_dists) out_dists = nullptr;
    const bool want_d = out_dists || keep_dists;
    if (want_d) dd.alloc(static_cast<size_t>(c + 1) * m.vocab());
    else if (out_logits) lg.alloc(static_cast<size_t>(c + 1) * m.vocab());
    // rows [L-1, L+c): one forward, or (forward_batch has no row cap, model.cpp:37-53) consecutive
    // <= 256-row forwards — batch invariance makes each row bitwise the one-forward row
    const int cap = m.has_kv() ? std::min(kPrefillChunk, m.max_forward_tokens()) : c + 1;
    for (int p0 = L - 1; p0 < L + c;) {
        const int p1 = std::min(L + c, p0 + cap);
        const int first = std::min(lane.kv_len, p0);
        if (p1 == L + c) lane.set_state(L, c, lane.kv_len, p0, S.main);  // the last piece: L + c = p1
        else lane.set_state(p1, 0, lane.kv_len, p0, S.main);
        const size_t at = static_cast<size_t>(p0 - (L - 1)) * m.vocab();
        if (want_d) m.dists(lane, p1 - first, p1 - p0, dd.p + at, S.main);
        else if (out_logits) m.logits(lane, p1 - first, lg.p + at, S.main);
        else m.forward(lane, p1 - first, S.main);
        lane.kv_len = std::max(lane.kv_len, p1);
        p0 = p1;
    }
    DevBuf<int32_t> rows(c + 1);
    gather_rows_kernel<<<1, 256, 0, S.main>>>(lane.argmax.p, L - 1, c + 1, rows.p);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaMemcpyAsync(out_argmax, rows.p, (c + 1) * 4, cudaMemcpyDeviceToHost, S.main));
    if (out_dists)
        CUDA_CHECK(cudaMemcpyAsync(out_dists, dd.p, dd.bytes(), cudaMemcpyDeviceToHost, S.main));
    else if (out_logits)
        CUDA_CHECK(cudaMemcpyAsync(out_logits, lg.p, lg.bytes(), cudaMemcpyDeviceToHost, S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    if (const char* dbg = std::getenv("DBL_DEBUG_STATE_FILE")) {  // debugging: the lane's KV state per call
        if (FILE* f = std::fopen(dbg, "a")) {
            unsigned long long h = 0xcbf29ce484222325ull;
            for (int i = 0; i <= c; ++i) h = (h ^ static_cast<uint32_t>(out_argmax[i])) * 0x100000001b3ull;
            std::fprintf(f, "argmax=%016llx %s\n", h, m.debug_state_hash(lane, L - 1).c_str());
            std::fclose(f);
        }
    }
    for (int i = 0; i <= c; ++i)
        if (out_argmax[i] < 0) throw_runtime("degenerate distribution");
    if (keep_dists) *keep_dists = std::move(dd);
}

// retrieval_forward (speculation.cpp:54-66): lookup (if enabled) -> one forward_batch over ctx ⊕
// candidates -> accept_with_model, all rows staying on the device
RetrievalOut retrieval_forward(Model& m, DeviceStore* st, const int32_t* ctx, int L, int depth, double temperature,
                               DeviceRng* rng, bool use_retrieval, bool want_probs) {
    if (L <= 0) throw_invalid("lookup: empty context");
    RetrievalOut r;
    std::vector<int32_t> cands;
    if (use_retrieval) {
        if (!st) throw_invalid("retrieval_forward: a datastore is required with use_retrieval");
        if (st->device() != m.device()) throw_invalid("model and datastore must live on the same device");
        const int64_t off[2] = {0, L};
        const int32_t dep = depth;
        const int dc = std::max(depth, 1);
        std::vector<int32_t> cbuf(dc);
        int32_t n = 0, src = DBL_SRC_MISS, order = 0;
        DeviceGuard g(st->device());
        st->lookup_batch(1, off, ctx, &dep, dc, cbuf.data(), &n, &src, &order, 0);
        cands.assign(cbuf.begin(), cbuf.begin() + n);
        r.source = src;
    }
    const int c = static_cast<int>(cands.size());
    DeviceGuard g(m.device());
    std::vector<int32_t> am(c + 1);
    DevBuf<double> dd;
    forward_stateless(m, ctx, L, cands.data(), c, am.data(), nullptr, nullptr, &dd);
    AcceptOut a = accept_with_model_dev(dd.p, m.vocab(), c + 1, cands.data(), c, temperature, rng, want_probs);
    r.emitted = std::move(a.emitted);
    r.matched_len = a.matched_len;
    r.n_probs = a.n_probs;
    r.probs = std::move(a.probs);
    return r;
}

// ------------------------------------------------------------------------ forward profiling
void profile_forward(Model& m, int ctx_len, int rows, int iters, double* out) {
    if (ctx_len < 1 || rows < 1 || iters < 1) throw_invalid("profile_forward: bad arguments");
    DeviceGuard g(m.device());
    Streams S;
    Lane lane(m, ctx_len + rows + 16);
    LaneIO io(&lane);
    std::vector<int32_t> X(ctx_len + rows);
    for (size_t i = 0; i < X.size(); ++i) X[i] = static_cast<int32_t>((i * 7919 + 13) % m.vocab());
    io.sync_tokens(X, S.main);
    catch_up(lane, ctx_len - 1, S.main);
    lane.set_state(ctx_len, rows - 1, lane.kv_len, ctx_len - 1, S.main);
    for (int i = 0; i < 2; ++i) m.forward(lane, rows, S.main);  // warm-up
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    // pass 1: whole-forward time (no per-GEMM events)
    Timer t;
    const long long l0 = launch_counter();
    CUDA_CHECK(cudaEventRecord(t.a, S.main));
    for (int i = 0; i < iters; ++i) m.forward(lane, rows, S.main);
    CUDA_CHECK(cudaEventRecord(t.b, S.main));
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    const long long launches = launch_counter() - l0;
    // pass 2: per-GEMM CUDA events on the launching stream
    GemmProfiler prof;
    m.set_profiler(&prof);
    for (int i = 0; i < iters; ++i) m.forward(lane, rows, S.main);
    m.set_profiler(nullptr);
    CUDA_CHECK(cudaStreamSynchronize(S.main));
    double gemm_ms = 0.0, bytes = 0.0, lm_ms = 0.0, lm_bytes = 0.0;
    const size_t per_fwd = prof.bytes.size() / iters;
    for (size_t k = 0; k < prof.bytes.size(); ++k) {
        float ms = 0.f;
        CUDA_CHECK(cudaEventElapsedTime(&ms, prof.ev[2 * k], prof.ev[2 * k + 1]));
        gemm_ms += ms;
        bytes += prof.bytes[k];
        if (per_fwd && k % per_fwd == per_fwd - 1) { lm_ms += ms; lm_bytes += prof.bytes[k]; }
    }
    // SURVEY §8(d) algorithmic bytes per forward: streamed weights + KV read over the context and
    // appended for the new rows + the embedding rows gathered
    const double kv_emb = static_cast<double>(m.kv_bytes_per_token()) * (ctx_len + rows) +
                          static_cast<double>(m.embed_bytes_per_token()) * rows;
    out[0] = t.ms() / iters;                          // forward ms
    out[1] = gemm_ms / iters;                          // forward-kernel ms (event-timed launches)
    out[2] = bytes / iters + kv_emb;                   // algorithmic bytes per forward
    out[3] = static_cast<double>(per_fwd);             // GEMM launches per forward
    out[4] = static_cast<double>(launches) / iters;    // kernel launches per forward
    out[5] = static_cast<double>((rows + 15) / 16 * 16);  // token columns (tp)
    out[6] = lm_ms / iters;                            // LM-head GEMM ms
    out[7] = lm_bytes / iters;                         // LM-head GEMM bytes
}

}  // namespace dbl
