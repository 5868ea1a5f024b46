// Tensor-parallel target: N shards of one transformer driven as one Model.
//
// Shards are Transformers with tp_rank/tp_size (column-parallel QKV / gate|up, row-parallel O / down,
// vocab-parallel LM head; shard-exact init).  One forward = every shard's fwd_kernel running
// concurrently; they exchange O / down partial tiles and the LM-head argmax through each other's
// exchange buffers inside the kernel (fwd.cuh), so every shard ends the forward with the same
// residual stream and the same argmax rows — no NCCL call on the path.
//
// In-process group (this class): shards may sit on different GPUs (peer access over NVLink) or on the
// same GPU (two shards co-reside: fwd_kernel takes <= half an SM), which is how TP is tested on one
// B200.  The decoder's lane lives with shard 0; shards r >= 1 get a mirror of the lane's token
// buffer and cursor before every forward (a few KB over NVLink) and keep their own KV caches.
#pragma once
#include <memory>
#include <vector>

#include "transformer.cuh"

namespace dbl {

class TpTransformer final : public Model {
  public:
    TpTransformer(const dbl_transformer_config& cfg, const std::vector<int>& devices);
    ~TpTransformer() override;
    int device() const override { return devices_[0]; }
    int vocab() const override { return cfg_.vocab; }
    bool has_kv() const override { return true; }
    int64_t weight_bytes() const override { return shards_[0]->weight_bytes(); }  // per GPU
    int64_t kv_bytes_per_token() const override { return shards_[0]->kv_bytes_per_token(); }
    int64_t embed_bytes_per_token() const override { return shards_[0]->embed_bytes_per_token(); }
    std::unique_ptr<LaneCache> make_cache(int capacity) override;
    void forward(Lane& lane, int max_tokens, cudaStream_t s) override;
    void logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) override;
    int max_forward_tokens() const override { return shards_[0]->max_forward_tokens(); }
    std::string kind() const override { return "transformer-tp"; }
    int persistent_grids() const override {
        int k = 0;
        for (int d : devices_) k += d == devices_[0];
        return k;
    }
    int persistent_grids_on(int dev) const override {
        int k = 0;
        for (int d : devices_) k += d == dev;
        return k;
    }
    void set_profiler(GemmProfiler* p) override { shards_[0]->set_profiler(p); }
    void set_smem_budget(int bytes) override {
        for (auto& sh : shards_) sh->set_smem_budget(bytes);
    }
    int world() const { return static_cast<int>(shards_.size()); }
    Transformer& shard(int r) { return *shards_[static_cast<size_t>(r)]; }

  private:
    void run(Lane& lane, int max_tokens, float* logits, cudaStream_t s);
    dbl_transformer_config cfg_;
    std::vector<int> devices_;
    std::vector<std::unique_ptr<Transformer>> shards_;
};

}  // namespace dbl
