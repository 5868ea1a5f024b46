// Skinny "weights x tokens" GEMM on tcgen05 (swap-AB) — the verify-forward contraction.
//
//   D[n, t] = sum_k W[n, k] * X[t, k]      W: [n_out, K] bf16 (K-major, streamed once, TMA EVICT_FIRST)
//                                          X: [tp, K]    bf16 (the <= 256 padded token rows, L2-resident)
// The 128 weight rows of a tile are the UMMA M side and the padded tokens are N (16..256), so one
// tcgen05.mma.kind::f16 (M=128, N=tp, K=16) covers every token of the forward and the kernel is pure
// weight streaming.  Work is split stream-K style over a fixed grid (one CTA per SM): each CTA takes
// an equal range of the (tile, 64-wide k-block) sequence; tiles split across CTAs are combined by
// the last-arriving CTA in a FIXED contributor order.  The split depends only on (n_out, K, #SMs) —
// never on the token count — so every token column is bitwise identical whether the forward carries
// 1 row or 100 (batch invariance: AR and verify forwards agree exactly).
// Warp roles: 0 = TMA producer, 1 = TMEM allocator + MMA issuer, 2..5 = epilogue (TMEM lane quadrant
// = warp % 4).
#pragma once
#include <cuda.h>

#include <vector>

#include "common.cuh"

namespace dbl {

struct LaneState;

enum class Epi : int {
    StoreBF16 = 0,  // out[t][n] = bf16(acc)
    ResidAdd = 1,   // out[t][n] += acc           (fp32 residual stream)
    SiluMul = 2,    // rows interleaved per 32-lane quadrant as 16 gate | 16 up: out[t][f] = bf16(silu(g)*u)
    Argmax = 3,     // per-tile (max, lowest idx) partials over rows n < n_valid; optional fp32 logits
    StoreF32 = 4,   // out[t][n] = acc            (tests)
};

struct GemmArgs {
    int n_out, K, tp, n_valid;
    int n_tiles, kb_total;
    long long units;
    int stages;
    int l2_prefetch_units;  // weight k-blocks per CTA warmed into L2 before the grid-dependency wait
    long long next_units;   // next GEMM of the forward (0 = none): its unit count, grid, k-blocks,
    int next_grid, next_kb, next_prefetch;  // and the k-blocks per CTA to warm into L2
    unsigned long long* trace;  // optional per-CTA %globaltimer stamps [grid][4] (DBL_GEMM_TRACE)
    void* out;
    int ld_out;
    float* logits;
    int ld_logits;
    float2* amax_ws;  // [n_tiles][tp] (value, index bits)
    float* ws;        // stream-K partial slots [2 * grid][tp][128]
    int* counters;    // [n_tiles], zero between launches
    const struct LaneState* lane;  // Argmax logits rows: [0, L + c - start) only (nullable: tp rows)
};

struct GemmWorkspace {  // per decode lane (a lane's GEMMs are stream-ordered)
    DevBuf<float> partials;
    DevBuf<int> counters;
    DevBuf<float2> amax;
    int grid = 0, max_tp = 0, max_tiles = 0;
    void ensure(int grid, int max_tp, int max_tiles);
};

int num_sms(int device);
void gemm_prepare();  // set kernel attributes (call before stream capture)
CUtensorMap make_tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, int box_rows);
// a tiled weight image (launch_tile_weights) of `tiles` 128 x 64 tiles as [tiles * 128][64] rows of
// 128 B: box (64, 128) at row tile * 128 is one contiguous 16 KiB tile
CUtensorMap make_tmap_bf16_tiled(const void* ptr, uint64_t tiles);
CUtensorMap make_tmap_bf16_kblocks(const void* ptr, uint64_t rows, uint64_t cols, int box_rows, int box_kb);

// Launch one GEMM.  tmW: weights (box 128 x 64), tmX: activations (box 16 x 64).
// DBL_GEMM_TRACE=1: every GEMM launch records per-CTA %globaltimer stamps (resident, dependency
// resolved, last load issued, epilogue done) — a device timeline without nsys (tools/gemm_timeline.py)
constexpr int kTraceLaunches = 4096, kTraceCtas = 320;
struct GemmTrace {
    DevBuf<unsigned long long> buf;
    int n = 0;
    std::vector<int> grid;
    std::vector<long long> bytes;
};
GemmTrace& gemm_trace();

struct GemmNext {  // the GEMM that follows in the forward (its first weight tiles are L2-warmed)
    const CUtensorMap* tmap;
    int n_out, K;
};
void gemm_launch(Epi epi, const CUtensorMap& tmW, const CUtensorMap& tmX, int n_out, int K, int tp,
                 int n_valid, void* out, int ld_out, float* logits, int ld_logits, GemmWorkspace& ws,
                 cudaStream_t s, const struct LaneState* lane = nullptr, const GemmNext* next = nullptr);
struct LaneState;
// final argmax over the per-tile partials: argmax[lane.start + t] for t in [0, L + c - start)
void argmax_finish(const GemmWorkspace& ws, int n_tiles, int tp, const LaneState* lane, int32_t* argmax,
                   cudaStream_t s);

}  // namespace dbl
