// Device model interface shared by the table model (config 1) and the transformer (configs 2-5).
// A model's forward reads a lane's token buffer and writes per-position argmax rows — the
// forward_batch contract (model.cpp:37-53) with greedy consumption (argmax_token, model.cpp:70-81).
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "lane.cuh"

namespace dbl {

// Per-(model, lane) mutable device state (KV cache for transformers; empty for tables).
struct LaneCache {
    virtual ~LaneCache() = default;
};

class Lane;

// Shared memory per forward CTA.  Two CTAs co-reside on an SM (a DOUBLE round's draft and target
// forwards, each a persistent grid): their sum must stay within the SM's 228 KB minus 1 KB per CTA.
// The target streams most of the bytes and needs the deeper ring at > 16 token columns (measured: 4 ->
// 6 stages at 32 columns saved 0.3 ms on Qwen3-14B at 16 tokens); the draft keeps 4 stages (3 cost it
// +3 %, profiles/r2af_*).
constexpr int kFwdSmemBudget = 136 * 1024;       // a model's default (the target role)
constexpr int kFwdSmemDraftBudget = 90 * 1024;   // the draft role beside a target (DoubleEngine)
constexpr int kFwdSmemSharedBudget = 113 * 1024; // both roles on one model (self-drafting)

// Optional per-GEMM CUDA-event timing of a model's forwards (bench roofline; off in the decode loop)
struct GemmProfiler {
    std::vector<cudaEvent_t> ev;  // pairs (before, after) per GEMM launch
    std::vector<double> bytes;    // algorithmic bytes of each timed GEMM (weights + activations)
    size_t used = 0;
    cudaEvent_t next(cudaStream_t s) {
        if (used == ev.size()) {
            cudaEvent_t e;
            CUDA_CHECK(cudaEventCreate(&e));
            ev.push_back(e);
        }
        cudaEvent_t e = ev[used++];
        CUDA_CHECK(cudaEventRecord(e, s));
        return e;
    }
    ~GemmProfiler() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

class Model {
  public:
    virtual ~Model() = default;
    virtual int device() const = 0;
    virtual int vocab() const = 0;
    virtual bool has_kv() const = 0;
    virtual int64_t weight_bytes() const { return 0; }
    // HBM bytes per context position a forward reads from the KV cache (and appends per new row)
    virtual int64_t kv_bytes_per_token() const { return 0; }
    virtual int64_t embed_bytes_per_token() const { return 0; }
    virtual std::unique_ptr<LaneCache> make_cache(int capacity) = 0;
    // a lane's cache when the lane goes away (models may keep a few for the next make_cache)
    virtual void recycle_cache(std::unique_ptr<LaneCache>) {}
    // Enqueue one forward on stream s: process positions [min(kv_len,row0), L+c) of the lane, write
    // lane.argmax[p] for those positions and set lane.start / lane.kv_len = L+c.  `max_tokens` is a
    // host-side upper bound of L+c-start (kernel shape bucket); the exact count is read on device.
    virtual void forward(Lane& lane, int max_tokens, cudaStream_t s) = 0;
    // Like forward, and also write fp32 logits (tables: probabilities) of rows [row0, L+c), in
    // order, to out_dev ((L+c-row0) x vocab).
    virtual void logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) = 0;
    // Like forward, and also write the fp64 next-token distributions of rows [row0, L+c), in order,
    // to out_dev ((L+c-row0) x vocab, at most max_rows): the ProbVector rows of forward_batch
    // (model.cpp:37-53) the sampled (temperature > 0) loop consumes.  Default: softmax of logits.
    virtual void dists(Lane& lane, int max_tokens, int max_rows, double* out_dev, cudaStream_t s);
    virtual int max_forward_tokens() const { return 1 << 30; }
    // One forward over several lanes at once (independent sequences sharing one weight stream): lane
    // b's rows [min(kv_len, row0), L+c) as in forward(); max_tokens bounds the rows of all lanes.
    virtual void forward_lanes(const std::vector<Lane*>& lanes, int max_tokens, cudaStream_t s);
    // dists() over several lanes in one forward (lane b's rows to outs[b], at most max_rows[b])
    virtual void dists_lanes(const std::vector<Lane*>& lanes, int max_tokens, const std::vector<int>& max_rows,
                             const std::vector<double*>& outs, cudaStream_t s);
    // persistent (all-SM, cooperatively launched) grids one forward places on device(): at most two may
    // co-run on a GPU, so the decoder serializes draft and target work when the sum would exceed it
    virtual int persistent_grids() const { return 0; }
    // persistent grids one forward places on GPU `dev` (tensor-parallel shards may span several GPUs)
    virtual int persistent_grids_on(int dev) const { return dev == device() ? persistent_grids() : 0; }
    virtual void set_profiler(GemmProfiler*) {}
    // debugging: hashes of the lane's device state (KV per layer for positions < upto, scratch buffers)
    virtual std::string debug_state_hash(Lane&, int /*upto*/) { return ""; }
    // shared memory per forward CTA (persistent forwards: fwd.cuh kFwdSmem*Budget)
    virtual void set_smem_budget(int /*bytes*/) {}
    // the draft beside a target on one GPU: forwards on 1/div of the SMs, launched plainly (1 = own grid)
    virtual void set_draft_grid(int /*div*/) {}
    virtual std::string kind() const = 0;
};

// A model's working buffers for one decode role.
class Lane {
  public:
    Lane(Model& m, int capacity);
    ~Lane();
    Model& model;
    int capacity;                 // token capacity of buf / argmax
    DevBuf<int32_t> buf, argmax;
    LaneState* state = nullptr;   // device
    std::unique_ptr<LaneCache> cache;
    DevBuf<float> logit_scratch;  // fp32 logits behind Model::dists (grown on demand)
    // host-side mirror (kept exact by the orchestrator)
    std::vector<int32_t> mirror;  // tokens the device buffer holds in [0, mirror.size())
    int kv_len = 0;               // host view of the valid KV prefix
    void set_state(int L, int c, int kv, int row0, cudaStream_t s);
};

}  // namespace dbl
