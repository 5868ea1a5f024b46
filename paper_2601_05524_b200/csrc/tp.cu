#include "tp.cuh"

namespace dbl {
struct TpComm::Impl {};
TpComm::TpComm(void*, int, int, int) : impl_(nullptr) { throw_runtime("tensor parallel exchange not available yet"); }
TpComm::~TpComm() { delete impl_; }
void TpComm::allreduce_add(const float*, int, int, float*, cudaStream_t) {}
void TpComm::argmax_combine(const GemmWorkspace&, int, int, int, const LaneState*, int32_t*, cudaStream_t) {}
void TpComm::gather_logits(float*, int, int, int, cudaStream_t) {}
}  // namespace dbl
