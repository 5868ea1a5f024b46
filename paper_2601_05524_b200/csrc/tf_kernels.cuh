// Transformer set-up kernels: seeded random init of every weight tensor and the tiled weight images the
// stream forward (fwd.cu) reads; plus the KV page / attention chunk constants it shares.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "lane.cuh"

namespace dbl {

constexpr int kPage = 64;       // KV page (tokens)
constexpr int kAttnChunk = 64;  // keys per split-KV chunk = one page (fixed => batch invariant)

// weights ~ N(0, std) from (seed, tensor, logical index); rows [r0, r0+rows) x cols [c0, c0+cols) of a
// logical [R, C] tensor written to dst (row stride ld)
void launch_init_normal(__nv_bfloat16* dst, int rows, int cols, int ld, uint64_t seed, uint64_t tensor,
                        int64_t r0, int64_t c0, int64_t C, float std, cudaStream_t s);
// gate/up fused layout: physical row p of the [2*ffn_local, h] block, interleaved 16 gate | 16 up per 32
void launch_init_gateup(__nv_bfloat16* dst, int ffn_local, int hidden, uint64_t seed, uint64_t gate_id,
                        uint64_t up_id, int64_t f0, float std, cudaStream_t s);
// fused [q; k; v] rows (q rows from rq0, k/v rows from rkv0 of the logical tensors), head rows permuted
// so that RoPE partners d, d + hd/2 sit in lanes l, l ^ 16 of one warp (fwd.cuh)
void launch_init_qkv(__nv_bfloat16* dst, int q_dim, int kv_dim, int hd, int hidden, uint64_t seed, uint64_t q_id,
                     uint64_t k_id, uint64_t v_id, int64_t rq0, int64_t rkv0, float std, cudaStream_t s);
// logical dim held by physical row pr of a head (the permutation above)
inline int qkv_perm_dim(int pr, int hd) {
    const int w = pr / 32, l = pr % 32;
    return l < 16 ? 16 * w + l : hd / 2 + 16 * w + l - 16;
}
void launch_fill(__nv_bfloat16* dst, int64_t n, float v, cudaStream_t s);
// row-major [rows][K] -> the stream forward's tiled weight image: 128 x 64 tiles, each one contiguous
// 16 KiB block, tile (m, kb) at ((m * K/64) + kb) * 8192 elements; rows padded to a multiple of 128
// with zeros.  (K % 64 == 0.)  Inverse: launch_untile_weights.
constexpr int kWTileRows = 128, kWTileK = 64;
inline int64_t tiled_rows(int64_t rows) { return (rows + kWTileRows - 1) / kWTileRows * kWTileRows; }
void launch_tile_weights(__nv_bfloat16* dst, const __nv_bfloat16* src, int rows, int K, cudaStream_t s);
void launch_untile_weights(__nv_bfloat16* dst, const __nv_bfloat16* src, int rows, int K, cudaStream_t s);

}  // namespace dbl
