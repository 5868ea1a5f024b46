// Random-init bf16 decoder-only transformer on sm_100a (configs 2-5): see transformer.cu.
#pragma once
#include <mutex>

#include "model.cuh"

namespace dbl {

class Transformer final : public Model {
  public:
    Transformer(const dbl_transformer_config& cfg, int device, void* nccl_comm);
    ~Transformer() override;
    int device() const override { return device_; }
    int vocab() const override { return cfg_.vocab; }
    bool has_kv() const override { return true; }
    int64_t weight_bytes() const override;
    int64_t kv_bytes_per_token() const override;
    int64_t embed_bytes_per_token() const override { return static_cast<int64_t>(cfg_.hidden) * 2; }
    std::unique_ptr<LaneCache> make_cache(int capacity) override;
    void recycle_cache(std::unique_ptr<LaneCache> c) override;
    void forward(Lane& lane, int max_tokens, cudaStream_t s) override;
    void logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) override;
    void forward_lanes(const std::vector<Lane*>& lanes, int max_tokens, cudaStream_t s) override;
    void dists_lanes(const std::vector<Lane*>& lanes, int max_tokens, const std::vector<int>& max_rows,
                     const std::vector<double*>& outs, cudaStream_t s) override;
    int max_forward_tokens() const override;
    std::string kind() const override { return "transformer"; }
    int persistent_grids() const override { return 1; }
    void set_smem_budget(int bytes) override;
    void set_draft_grid(int div) override;
    std::string debug_state_hash(Lane& lane, int upto) override;
    void set_profiler(GemmProfiler* p) override;
    void get_weight(const std::string& name, int layer, uint16_t* out, int64_t numel);
    int tp_rank() const { return cfg_.tp_rank; }
    int tp_size() const { return cfg_.tp_size < 1 ? 1 : cfg_.tp_size; }
    // one forward over explicit lane pieces (a tensor-parallel shard's mirror of the decoder's lane)
    void forward_raw(LaneState* state, const int32_t* buf, int32_t* argmax, LaneCache* cache, int max_tokens,
                     float* logits_dev, cudaStream_t s);
    // tensor parallel: make every rank's lane cache address all ranks' exchange buffers (rank order)
    static void link_tp(const std::vector<LaneCache*>& caches);
    // tensor parallel with one process per shard: export this shard's exchange buffers as 4 CUDA IPC
    // handles (out: 4 x cudaIpcMemHandle_t), then import every rank's (rank order, world x 4) — after
    // which every lane cache of this shard exchanges with the other processes inside fwd_kernel
    void ipc_export(void* out);
    void ipc_import(const void* all, int world);
    // the same model-level exchange state for shards of ONE process (TpTransformer)
    static void link_models(const std::vector<Transformer*>& shards);
    // tensor-parallel shards sharing one GPU: each forward takes 1/k of the SMs (set before make_cache)
    void set_shards_per_device(int k) { shards_per_device_ = k; }

    struct Impl;
    static int64_t weight_bytes_of(const Impl& m);
    void ensure_xbuf();  // this shard's model-level exchange buffers (allocated once)

  private:
    Impl* impl_ = nullptr;
    dbl_transformer_config cfg_;
    int device_;
    int shards_per_device_ = 1;
    // lane caches (KV, scratch, phase table: ~100s of MB of allocations) kept for reuse across run()
    // calls — every public call builds fresh lanes, and re-allocating them dominated its host overhead
    std::mutex pool_mu_;
    std::vector<std::unique_ptr<LaneCache>> pool_;
};

}  // namespace dbl
