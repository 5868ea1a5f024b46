// In-process tensor-parallel group (tp.cuh).
#include "tp.cuh"

#include "fwd.cuh"

namespace dbl {

namespace {
struct ShardLane {  // a shard's mirror of the decoder's lane + its own KV cache
    int device = 0;
    DevBuf<int32_t> buf, argmax;
    DevBuf<LaneState> state;
    std::unique_ptr<LaneCache> cache;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    ~ShardLane() {
        if (stream) {
            cudaSetDevice(device);
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
        if (done) cudaEventDestroy(done);
    }
};

struct TpCache final : LaneCache {
    int capacity = 0;
    std::unique_ptr<LaneCache> c0;                  // shard 0's cache (the decoder's lane)
    std::vector<std::unique_ptr<ShardLane>> rest;  // shards 1..N-1
    cudaEvent_t ready = nullptr;
    ~TpCache() override {
        rest.clear();
        if (ready) cudaEventDestroy(ready);
    }
};
}  // namespace

TpTransformer::TpTransformer(const dbl_transformer_config& cfg, const std::vector<int>& devices)
    : cfg_(cfg), devices_(devices) {
    const int world = static_cast<int>(devices.size());
    if (world < 2 || world > kMaxTpRanks) throw_invalid("tensor parallel: 2..8 shards");
    cfg_.tp_size = world;
    for (int r = 0; r < world; ++r) {  // peer access between distinct devices (NVLink)
        for (int q = 0; q < world; ++q) {
            if (devices[r] == devices[q]) continue;
            DeviceGuard g(devices[r]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_CHECK(e);
            cudaGetLastError();
        }
    }
    for (int r = 0; r < world; ++r) {
        dbl_transformer_config c = cfg_;
        c.tp_rank = r;
        shards_.push_back(std::make_unique<Transformer>(c, devices[r], nullptr));
        int same = 0;
        for (int q = 0; q < world; ++q) same += devices[q] == devices[r];
        shards_.back()->set_shards_per_device(same);
    }
    std::vector<Transformer*> ptrs;
    for (auto& s : shards_) ptrs.push_back(s.get());
    Transformer::link_models(ptrs);  // model-level exchange buffers + exchange-tag counter
}

TpTransformer::~TpTransformer() = default;

std::unique_ptr<LaneCache> TpTransformer::make_cache(int capacity) {
    auto tc = std::make_unique<TpCache>();
    tc->capacity = capacity;
    tc->c0 = shards_[0]->make_cache(capacity);
    for (int r = 1; r < world(); ++r) {
        auto sl = std::make_unique<ShardLane>();
        sl->device = devices_[r];
        DeviceGuard g(sl->device);
        sl->buf.alloc(capacity);
        sl->argmax.alloc(capacity);
        sl->state.alloc(1);
        sl->buf.zero();
        sl->state.zero();
        sl->cache = shards_[r]->make_cache(capacity);
        int lo = 0, hi = 0;
        CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_CHECK(cudaStreamCreateWithPriority(&sl->stream, cudaStreamNonBlocking, hi));
        CUDA_CHECK(cudaEventCreateWithFlags(&sl->done, cudaEventDisableTiming));
        tc->rest.push_back(std::move(sl));
    }
    {
        DeviceGuard g(devices_[0]);
        CUDA_CHECK(cudaEventCreateWithFlags(&tc->ready, cudaEventDisableTiming));
        CUDA_CHECK(cudaDeviceSynchronize());
    }
    return tc;
}

void TpTransformer::run(Lane& lane, int max_tokens, float* logits, cudaStream_t s) {
    TpCache& tc = *static_cast<TpCache*>(lane.cache.get());
    DeviceGuard g(devices_[0]);
    CUDA_CHECK(cudaEventRecord(tc.ready, s));
    // mirror the lane (tokens + cursor) to every other shard, then launch all shards together
    for (auto& sl : tc.rest) {
        DeviceGuard gs(sl->device);
        CUDA_CHECK(cudaStreamWaitEvent(sl->stream, tc.ready, 0));
        CUDA_CHECK(cudaMemcpyAsync(sl->buf.p, lane.buf.p, static_cast<size_t>(tc.capacity) * 4, cudaMemcpyDefault,
                                   sl->stream));
        CUDA_CHECK(cudaMemcpyAsync(sl->state.p, lane.state, sizeof(LaneState), cudaMemcpyDefault, sl->stream));
    }
    shards_[0]->forward_raw(lane.state, lane.buf.p, lane.argmax.p, tc.c0.get(), max_tokens, logits, s);
    for (size_t r = 0; r < tc.rest.size(); ++r) {
        ShardLane& sl = *tc.rest[r];
        DeviceGuard gs(sl.device);
        shards_[r + 1]->forward_raw(sl.state.p, sl.buf.p, sl.argmax.p, sl.cache.get(), max_tokens, logits, sl.stream);
        CUDA_CHECK(cudaEventRecord(sl.done, sl.stream));
    }
    for (auto& sl : tc.rest) CUDA_CHECK(cudaStreamWaitEvent(s, sl->done, 0));
}

void TpTransformer::forward(Lane& lane, int max_tokens, cudaStream_t s) { run(lane, max_tokens, nullptr, s); }

void TpTransformer::logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) {
    run(lane, max_tokens, out_dev, s);  // each shard writes its vocab columns of out_dev (peer stores)
}

}  // namespace dbl
