// Device TableModel (config 1): see table_model.cu.
#pragma once
#include "model.cuh"

namespace dbl {

constexpr int kMaxTableOrder = 16;

class TableModel final : public Model {
  public:
    TableModel(int order, int vocab, int64_t n_rows, const int32_t* windows, const double* probs,
               const double* fallback, int device);
    int device() const override { return device_; }
    int vocab() const override { return vocab_; }
    bool has_kv() const override { return false; }
    int64_t weight_bytes() const override { return n_rows_ * vocab_ * 8; }
    std::unique_ptr<LaneCache> make_cache(int) override { return nullptr; }
    void forward(Lane& lane, int max_tokens, cudaStream_t s) override;
    void logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) override;
    void dists(Lane& lane, int max_tokens, int max_rows, double* out_dev, cudaStream_t s) override;
    std::string kind() const override { return "table"; }

  private:
    void launch(Lane& lane, int max_tokens, float* probs_out, double* dist_out, cudaStream_t s);
    int device_, order_, vocab_, cap_mask_ = 0;
    int64_t n_rows_;
    DevBuf<int32_t> windows_, slots_;
    DevBuf<double> probs_, fallback_;
};

}  // namespace dbl
