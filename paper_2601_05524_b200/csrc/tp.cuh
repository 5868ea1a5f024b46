// Tensor-parallel exchange for the sharded target (row-parallel O/down partial sums, vocab-parallel
// argmax).  Deterministic by construction: partials are exchanged (pure data movement) and every
// rank sums them in rank order, so results do not depend on message size or arrival order.
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "lane.cuh"

namespace dbl {

class TpComm {
  public:
    TpComm(void* comm, int rank, int world, int device);
    ~TpComm();
    // resid[t][i] += sum_r partial_r[t][i]  (rank order), t < tp
    void allreduce_add(const float* partial, int tp, int h, float* resid, cudaStream_t s);
    // vocab-parallel argmax: combine per-rank (max, lowest global id) -> argmax[start + t]
    void argmax_combine(const GemmWorkspace& ws, int n_tiles, int tp, int vocab_offset, const LaneState* lane,
                        int32_t* argmax, cudaStream_t s);
    void gather_logits(float* logits, int tp, int vocab_l, int ld, cudaStream_t s);

  private:
    struct Impl;
    Impl* impl_;
};

}  // namespace dbl
