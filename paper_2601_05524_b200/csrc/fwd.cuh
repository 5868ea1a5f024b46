// The verify forward as ONE persistent, dependency-driven kernel ("stream forward").
//
// Why: a decode forward (M <= ~40 token rows) is pure weight streaming — 28 GB for Qwen3-14B — but
// as ~370 separate kernels every GEMM pays a pipeline ramp and drain, and the QKV -> attention -> O
// chain idles HBM for ~22 us per layer (profiles/r1_gemm_timeline.txt).  Here one CTA per SM runs
// the whole forward as a fixed list of phases:
//
//   EMBED | per layer: QKV(gemm) ATTN COMBINE O(gemm) GATE|UP(gemm) DOWN(gemm) | LM-HEAD(gemm) ARGMAX
//
// and the only thing that waits on a data dependency is the consumer side of the tensor core: the
// TMA producer streams every weight tile of the forward, phase after phase, into the shared-memory
// ring as soon as a slot frees; activation tiles (the B operand) are loaded when the phase they
// depend on has completed (a gpu-scope counter per phase, release/acquire).  While a CTA waits for
// attention or a split-K fixup, its ring is already filling with the next GEMM's weights.
//
// RMSNorm is folded: the residual-producing epilogues (embedding, O, down) write the fp32 residual,
// its bf16 copy (the next GEMM's B operand) and per-128-row sums of squares; the consuming GEMM's
// epilogue scales column t by rsqrt(mean(x_t^2) + eps) (norm weights are 1 in this random-init
// family and are folded into the projection).  Q/K RMSNorm + RoPE + the paged-KV append run in the
// QKV epilogue (each 128-row tile holds whole heads; rows are permuted at init so RoPE partners
// d, d + hd/2 sit in lanes l, l ^ 16 of one warp).
//
// Tensor parallel (tp_world > 1): QKV / gate|up are column-parallel and O / down row-parallel, so the
// O and down tiles are partial sums.  The tile's finisher pushes its partial into every rank's
// exchange slot (peer stores) and releases a per-(source, tile) flag at system scope; every rank then
// sums the ranks' partials in rank order — identical residual streams on all ranks, no NCCL call.
// The LM head is vocab-parallel; ranks exchange per-token (max, lowest global id) the same way.
//
// Batch invariance (the lossless identity with target-only AR) holds as in gemm.cu: every split /
// reduction order is a function of the model shape and the SM count, never of the token count.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "lane.cuh"

namespace dbl {

enum FwdPhaseKind : int { kPhEmbed = 0, kPhGemm = 1, kPhAttn = 2, kPhArgmax = 3, kPhCombine = 4 };
enum FwdEpi : int { kFeQkv = 0, kFeResid = 1, kFeSilu = 2, kFeLogits = 3 };

struct FwdPhase {
    int kind, epi;
    int wmap, xmap;      // FwdArgs::wmaps / xmaps index (weights box 128x64, activations boxes 4..64 x 64)
    int w_row0;          // first row of this phase's weights in its (all-layers) tensor map
    int n_out, K, n_tiles, kb;
    int units;           // n_tiles * kb (stream-K units; < 2^31 / #SMs, host-checked)
    int active, offset;  // CTAs taking part, rotated by offset (spreads small phases over SMs)
    int count;           // done[] increments per forward (GEMM: tiles; others: CTAs)
    int dep;             // phase whose completion gates this one (-1: none)
    int layer;
    // per-layer attention data (QKV / ATTN phases)
    __nv_bfloat16* kc;   // this layer's K cache [pages][nkv][64][hd]
    __nv_bfloat16* vc;
    const __nv_bfloat16* qn;  // q/k RMSNorm weights (nullable)
    const __nv_bfloat16* kn;
};

// Tensor parallel: every rank's exchange buffers, addressed directly (same device, peer device over
// NVLink, or an IPC mapping).  Written remotely, read locally.
constexpr int kMaxTpRanks = 8;
struct TpPeers {
    float* xch[kMaxTpRanks];                 // [parity][src rank][h/128 tiles][256 cols][128 rows] fp32 partials
    unsigned long long* xflag[kMaxTpRanks];  // [parity][src rank][h/128 tiles] tags (parity: O 0, down 1)
    float2* axch[kMaxTpRanks];               // [src rank][256] (max logit, global id) per token
    unsigned long long* aflag[kMaxTpRanks];  // [src rank] tags
};

// Batched forward (several independent sequences in one weight stream): lane b's
// rows [min(kv_len, row0), L + c) are rows off[b].. of the forward; every lane has its own token
// buffer, argmax rows, page table and KV cache (same capacity), addressed relative to lane 0's.
constexpr int kMaxBatch = 16;
struct FwdBatch {
    int n;  // 0: single-lane forward (FwdArgs::lane / buf / argmax / page_table)
    LaneState* lane[kMaxBatch];
    const int32_t* buf[kMaxBatch];
    int32_t* argmax[kMaxBatch];
    const int32_t* page_table[kMaxBatch];
    long long koff[kMaxBatch], voff[kMaxBatch];  // element offsets of lane b's K / V cache from lane 0's
    int* row_base;  // optional out: forward row of lane b's position p = row_base[b] + p (logits consumers)
};

struct FwdArgs {
    CUtensorMap wmaps[5];  // qkv, o, gate|up, down (all layers stacked), lm head
    CUtensorMap xmaps[3][5];  // xb, attn, act; boxes of 4, 8, 16, 32, 64 token rows
    const FwdPhase* ph;
    int n_ph;
    int dbg;               // DBL_FWD_DBG (experiments only; results invalid): 1 16 activation rows only, 3 watchdog test
    int tp, stages, nacc, acc_cols;
    LaneState* lane;
    const int32_t* buf;
    int32_t* argmax;
    const __nv_bfloat16* embed;
    int h, nh, nkv, hd, q_dim, kv_dim, ffn_l, vocab_l, max_chunks;
    float eps;
    float* resid;        // [256][h] fp32 residual stream
    __nv_bfloat16* xb;   // [256][h] bf16(resid): B operand of QKV / gate|up / LM head
    __nv_bfloat16* qbuf; // [256][nh][hd]
    __nv_bfloat16* attn; // [256][q_dim]
    __nv_bfloat16* act;  // [256][ffn_l]
    float* ssq;          // [h/128][256] per-tile sums of squares of the residual
    float* part_o;       // attention split-KV partials [256][nh][max_chunks][hd]
    float* part_ml;      // [256][nh][max_chunks][2]
    const float2* rope;  // [max_seq][hd/2] (cos, sin)
    int max_seq;
    const int32_t* page_table;
    float* ws;           // stream-K partial slots [2*G][tp][128]
    unsigned long long* slot_flag;  // [2*G] partial-slot flags: (epoch << 12 | phase + 1) when written
    float2* amax;        // LM-head per-tile (max, idx) [n_tiles][tp]
    float* logits;       // optional fp32 logits rows [T][ld_logits]
    int ld_logits;
    unsigned long long* done;   // [n_ph] monotone completion counters
    unsigned long long* epoch;  // forwards completed on this cache
    int* err;                   // watchdog: the tag of the aborted forward (fwd.cu), else stale / 0
    unsigned long long wd_ns;   // watchdog: a wait without progress for this long aborts the forward
    unsigned long long* trace;  // optional [n_ph][G][16] %globaltimer stamps
    int tp_world, tp_rank, vocab_off;  // tensor parallel (world 1: none); vocab_off = rank * vocab_l
    TpPeers peers;
    // optional model-level forward counter for the exchange tags (one process per shard: the exchange
    // buffers outlive lane caches, so their tags must not restart with a new cache); nullptr = epoch
    unsigned long long* tp_epoch;
    FwdBatch batch;
};
// the kernel takes FwdArgs by value: past 4 KiB of parameters the launch takes a slower parameter
// path (measured in r1h: +9-13 % on the whole forward)
static_assert(sizeof(FwdArgs) <= 4096, "FwdArgs must stay within 4 KiB of kernel parameters");

constexpr int kFwdThreads = 192;  // warp 0 TMA producer, warp 1 MMA, warps 2..5 epilogue / aux work
constexpr int kFwdMiscBytes = 16 * 1024;     // static shared state (barriers, reductions, attention);
                                             // <= 16 KiB keeps 2 ring stages at 256 token columns
constexpr int kFwdMaxStages = 24;
// shared-memory budgets per forward CTA: model.cuh (kFwdSmem*Budget)
constexpr int kFwdMinUnits = 4;             // smallest stream-K range worth a CTA (4 x 16 KiB)

void fwd_prepare();  // kernel attributes (call once, outside graph capture)
// stages for a token-column bucket; smem bytes returned through *smem
int fwd_stages(int tp, int budget, size_t* smem);

void fwd_launch(const FwdArgs& a, int grid, size_t smem, cudaStream_t s, bool coop = true);

// DBL_FWD_TRACE=1: every forward records per-(phase, CTA) %globaltimer stamps — [0] first weight tile
// issued, [1] activation dependency resolved (producer), [2] last contribution signalled, [3] epilogue
// start, [4] first MMA, [5] last MMA, [6] epilogue done — into one buffer [n_ph][grid][8] (overwritten
// by each forward); tools/fwd_timeline.py reads it back.
unsigned long long* fwd_trace_buffer(int n_ph, int grid);  // nullptr unless tracing
void fwd_trace_read(unsigned long long* dst, long long cap, int* n_ph, int* grid);

}  // namespace dbl
