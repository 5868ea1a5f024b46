#include "transformer.cuh"
namespace dbl {
struct Transformer::Impl {};
Transformer::Transformer(const dbl_transformer_config& cfg, int device, void*) : cfg_(cfg), device_(device) {
    throw_runtime("transformer: not built yet");
}
Transformer::~Transformer() { delete impl_; }
int64_t Transformer::weight_bytes() const { return 0; }
std::unique_ptr<LaneCache> Transformer::make_cache(int) { return nullptr; }
void Transformer::forward(Lane&, int, cudaStream_t) {}
void Transformer::logits(Lane&, int, float*, cudaStream_t) {}
int Transformer::max_forward_tokens() const { return 256; }
void Transformer::get_weight(const std::string&, int, uint16_t*, int64_t) {}
}  // namespace dbl
