// K3' — the sampled (temperature > 0) decode path: acceptance, verification and correction kernels
// over per-position fp64 distributions, consuming the reference's derive_rng streams draw for draw.
#pragma once
#include <cstdint>

#include "model.cuh"
#include "verify.cuh"

namespace dbl {

// lane error codes written by the sampled kernels (LaneState::error / RoundResult::*_error)
enum SampleErr : int { kSampDegenerate = 1, kSampCapacity = 2, kSampInvalid = 3, kSampResidualZero = 4 };
[[noreturn]] void raise_sample_error(int code);
// wide vocabularies on the reference-exact path (sequential fp64 sums and scan, fp64 pow) on every device
void set_exact_sampling(bool on);

// fp32 logits rows -> fp64 softmax rows of positions [row0, L+c) of `lane`; logits row of position p is
// p - start (single-lane forward) or *row_base + p (batched forward)
void launch_softmax_rows(const float* logits, const LaneState* lane, int vocab, double* out, int max_rows,
                         const int* row_base, cudaStream_t s);
// Rng(seed) into g[0]
void launch_seed_rng(DevRng* g, uint64_t seed, cudaStream_t s);
// g[lane] = derive_rng(seed, round, lane) for lane in {0, 1, 2} (rng_d, rng_t, rng_v; pipeline.cpp:227-231)
void launch_derive_rngs(DevRng* g, uint64_t seed, uint64_t round, cudaStream_t s);

// one draft segment (accept_with_model at T > 0, speculation.cpp:7-52) over dist rows of positions
// [row0, L+c); the eff rows of the emitted tokens are appended to chain (row (L - L0) + i), so the
// chain's probs stay aligned with its tokens (iterative_draft, speculation.cpp:76-84)
void launch_draft_accept_sampled(Lane& lane, RoundResult* rr, int seg, int L0, const double* dist, double* chain,
                                 int chain_cap, DevRng* rng_d, double temperature, double* scratch, cudaStream_t s);
// the target side of a round: finish_round's verification of the speculative tail against
// tempered target rows with rng_v (+ residual_sample correction, pipeline.cpp:110-140) and the
// target's own accept_with_model over its candidates with rng_t (pipeline.cpp:64-67).  serial = the
// run_serial_sd variant: no candidates, the bonus token is sample(dists.back(), rng_v)
// (harness.cpp:283-330).  scratch: 3 rows of vocab doubles.
void launch_target_accept_sampled(Lane& lane, int n_committed, RoundResult* rr, const double* dist,
                                  const double* spec_probs, DevRng* rng_t, DevRng* rng_v, double temperature,
                                  bool serial, double* scratch, cudaStream_t s);
// one run_vanilla_ar step at T > 0 (harness.cpp:239-241): sample(dist, rng) and append
void launch_ar_sample(Lane& lane, const double* dist, DevRng* rng, double temperature, double* scratch,
                      int32_t* out_host, int i, cudaStream_t s);

}  // namespace dbl
