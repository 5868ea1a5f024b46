#pragma once
#include "model.cuh"

namespace dbl {
void launch_draft_accept(Lane& lane, RoundResult* rr_dev, int seg, cudaStream_t s);
void launch_target_accept(Lane& lane, int n_committed, RoundResult* rr_dev, cudaStream_t s);
}  // namespace dbl
