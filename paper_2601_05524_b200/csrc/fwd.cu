// The persistent stream-forward kernel (design: fwd.cuh).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "fwd.cuh"
#include "sm100.cuh"
#include "tf_kernels.cuh"

namespace dbl {

namespace {

using namespace sm100;

constexpr int kBM = 128, kBK = 64;
constexpr int kABytes = kBM * kBK * 2;  // one 128 x 64 bf16 weight tile
constexpr int kBatch = 2;               // split-K partials: 2 contributors x 16 columns of loads in flight

// ------------------------------------------------------------------ small helpers
// Watchdog: a wait that makes no progress for a.wd_ns (a missing tensor-parallel peer, a host contract
// violation) aborts the forward instead of trapping: the first stuck thread writes the forward's tag
// (epoch-derived, so a later forward ignores it) into a.err, every other wait sees it within 128
// polls and gives up, the kernel drains its in-flight copies and MMAs and exits, and the argmax rows
// come back as -1 (a degenerate row: the API raises runtime_error).  The CUDA context stays usable.
__shared__ int g_wdtag;  // this forward's abort tag (set at kernel start from the lane's epoch)
__device__ __forceinline__ int wd_tag(const FwdArgs&) { return g_wdtag; }
__device__ __forceinline__ bool aborted(const FwdArgs& a) {
    return *reinterpret_cast<volatile int*>(a.err) == wd_tag(a);
}
__device__ __noinline__ void watchdog_fire(const FwdArgs& a, int code, int phase) {
    if (atomicExch(a.err, wd_tag(a)) != wd_tag(a))
        printf("dbl fwd_kernel watchdog: CTA %d thread %d stuck (role %d, phase %d): forward aborted\n", blockIdx.x,
               threadIdx.x, code, phase);
}
struct Spin {
    unsigned long long t0 = 0;
    unsigned n = 0;
    // true: give up (this forward was aborted)
    __device__ __forceinline__ bool tick(const FwdArgs& a, int code, int phase) {
        if ((++n & 127u) == 0) {
            if (aborted(a)) return true;
            const unsigned long long t = globaltimer();
            if (!t0) {
                t0 = t;
            } else if (t - t0 > a.wd_ns) {
                watchdog_fire(a, code, phase);
                return true;
            }
        }
        return false;
    }
};
__device__ __forceinline__ bool mbar_wait_wd(uint64_t* bar, uint32_t par, const FwdArgs& a, int code, int phase) {
    Spin s;
    while (!mbar_try(bar, par))
        if (s.tick(a, code, phase)) return true;
    return false;
}

// A phase's stream-K split: phase-local CTA ci takes units [ci*U/A, (ci+1)*U/A).  Unit counts fit in
// 32 bits (host-checked); products are formed in 64 bits once per phase, never in the per-tile loops.
struct Range {
    int b0, b1;
    int ci;  // phase-local CTA index
};
__device__ __forceinline__ int range_begin(int ci, int U, int A) { return ci * U / A; }  // ci*U < 2^31
__device__ __forceinline__ Range cta_range(const FwdPhase& P, int c, int G) {
    int ci = c - P.offset;
    if (ci < 0) ci += G;
    Range r{0, 0, ci};
    if (ci < P.active) {
        r.b0 = range_begin(ci, P.units, P.active);
        r.b1 = range_begin(ci + 1, P.units, P.active);
    }
    return r;
}
// phase-local CTA whose range contains unit u: largest ci with floor(ci U / A) <= u
__device__ __forceinline__ int owner_of(int u, int U, int A) { return ((u + 1) * A - 1) / U; }

__device__ __forceinline__ bool dep_ok(const FwdArgs& a, int p, unsigned long long ep) {
    if (p < 0) return true;
    if (a.dbg == 3 && p == a.n_ph / 2) return false;  // DBL_FWD_DBG=3: a dependency that never resolves (watchdog test)
    if (ld_relaxed_u64(a.done + p) < (ep + 1) * static_cast<unsigned long long>(a.ph[p].count)) return false;
    fence_acq_rel_gpu();
    return true;
}
__device__ __forceinline__ bool wait_dep(const FwdArgs& a, int p, unsigned long long ep, int code) {
    Spin s;
    while (!dep_ok(a, p, ep))  // each probe is an L2 round trip
        if (s.tick(a, code, p)) return true;
    return false;
}
__device__ __forceinline__ void stamp(const FwdArgs& a, int p, int k) {
    if (a.trace) a.trace[(static_cast<long long>(p) * gridDim.x + blockIdx.x) * 16 + k] = globaltimer();
}

// GEMM unit cursor: the (phase, unit) sequence of this CTA over the whole forward.  Advanced
// incrementally — the single-threaded producer and MMA loops must not divide (a 64-bit division is a
// ~150-instruction subroutine; one per 16 KiB tile caps a CTA at a fraction of its HBM share).
struct Cur {
    int p;         // phase (n_ph = exhausted)
    int u, e;      // unit, end of this CTA's range
    int m, kb;     // tile row and k-block of u
    int KB, wrow, wmap, xmap, dep;  // the phase's fields
};
__device__ __forceinline__ void seek(Cur& k, const FwdArgs& a, int c, int G) {
    for (; k.p < a.n_ph; ++k.p) {
        const FwdPhase& P = a.ph[k.p];
        if (P.kind != kPhGemm) continue;
        const Range r = cta_range(P, c, G);
        if (r.b0 < r.b1) {
            k.u = r.b0;
            k.e = r.b1;
            k.KB = P.kb;
            k.m = r.b0 / P.kb;
            k.kb = r.b0 - k.m * P.kb;
            k.wrow = P.w_row0;
            k.wmap = P.wmap;
            k.xmap = P.xmap;
            k.dep = P.dep;
            return;
        }
    }
}
__device__ __forceinline__ void step(Cur& k, const FwdArgs& a, int c, int G) {
    ++k.u;
    if (++k.kb == k.KB) {
        k.kb = 0;
        ++k.m;
    }
    if (k.u >= k.e) {
        ++k.p;
        seek(k, a, c, G);
    }
}
struct Ring {  // ring slot + mbarrier parity of the next use
    int st = 0;
    uint32_t ph = 0;
    __device__ __forceinline__ void next(int S) {
        if (++st == S) {
            st = 0;
            ph ^= 1u;
        }
    }
};

// Small, cold inputs of the epilogue / attention chains (norm weights, RoPE rows, embedding rows, the
// context's KV cache) would otherwise be fetched from DRAM at the moment they are needed — behind a
// saturated weight stream, i.e. microseconds per dependent load.  They are warmed into L2 ahead of use
// with bulk prefetches, split over `parts` issuers.
__device__ __forceinline__ void l2_warm(const void* base, long long bytes, int part, int parts) {
    constexpr long long kChunk = 16384;
    const long long n = (bytes + kChunk - 1) / kChunk;
    const uintptr_t b = reinterpret_cast<uintptr_t>(base) & ~uintptr_t(15);
    const long long end = static_cast<long long>(reinterpret_cast<uintptr_t>(base) + bytes);
    for (long long i = part; i < n; i += parts) {
        const long long lo = static_cast<long long>(b) + i * kChunk;
        const long long len = std::min<long long>(kChunk, end - lo);
        if (len > 0) l2_prefetch_bulk(reinterpret_cast<const void*>(lo), static_cast<uint32_t>((len + 15) & ~15LL));
    }
}

// the embedding gather's range check (the table covers the unsharded vocab: vocab_l per rank)
__device__ __forceinline__ bool valid_token(int tok, const FwdArgs& a) {
    return static_cast<unsigned>(tok) < static_cast<unsigned>(a.vocab_l * a.tp_world);
}

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// 32 columns x 32 lanes -> lane l holds the sum over the warp's lanes of column l (fixed tree)
__device__ __forceinline__ float warp_colsum32(float (&v)[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool hi = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const float send = hi ? v[i] : v[i + s];
            const float keep = hi ? v[i + s] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return v[0];
}

// Split-KV causal attention, one (kv head, 64-key chunk, token block) item per CTA: the 4 aux warps
// load the chunk's K and V rows and the block's q rows (all G q heads of the kv head x up to Tb
// tokens: R = G * Tb <= 16 rows, one m16 tile) together — one round trip — then run scores and P*V
// on the tensor cores (mma.sync m16n8k16 bf16 -> fp32: warp w takes keys [16w, 16w + 16) of the
// scores and head dims [w HD/4, (w + 1) HD/4) of the output), the per-row softmax in fp32 (one warp
// per row, fixed butterflies).  A position's chunk partials are combined by the next phase
// (ATTN_COMBINE: one warp per (token, q head), chunks in order).  Every row's arithmetic is a
// function of its position only — a tensor-core dot product never depends on the other rows — so
// the result is the same however many tokens the forward carries (batch invariance).
constexpr int kAttnRows = 16;
constexpr int kQStride = 128 + 8;         // bf16 per q row (padded: conflict-free fragment loads)
constexpr int kPStride = kAttnChunk + 4;  // fp32 per probability row (padded likewise)
struct alignas(16) AttnSmem {
    __nv_bfloat16 q[kAttnRows * kQStride];  // q rows of the item (row r = token tt * G + head hh)
    float p[kAttnRows * kPStride];          // scores, then probabilities
    float m[kAttnRows], l[kAttnRows];       // per-row max and sum of this chunk
};

// tokens per attention item: all G = nh / nkv q heads of a kv head x Tb tokens fill <= kAttnRows rows
__device__ __forceinline__ int attn_block(const FwdArgs& a) { return max(1, kAttnRows / (a.nh / a.nkv)); }

// opaque copy: values derived from it are not hoisted out of the forward's phase loop (attention-only
// quantities would otherwise stay live through the GEMM epilogues and push them into local memory)
__device__ __forceinline__ int opaque(int x) {
    int y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

// D += A * B, m16n8k16, bf16 inputs, fp32 accumulate (fragment layouts: PTX ISA, mma.m16n8k16)
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

template <int HD>
__device__ __forceinline__ void attn_item(const FwdArgs& a, AttnSmem& S, int g, int j, int t0, int nt, int pos0,
                                          const int32_t* page_table, const __nv_bfloat16* kc,
                                          const __nv_bfloat16* vc, int ph) {
    constexpr int KS = HD / 16;  // k-steps of the scores
    constexpr int NP = HD / 64;  // pairs of n8 output tiles per warp (HD / 4 dims per warp)
    const int et = opaque(static_cast<int>(threadIdx.x)) - 64, ew = et >> 5, lane = et & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int nh = opaque(a.nh), nkv = opaque(a.nkv), Gq = nh / nkv;
    const int k0 = j * kAttnChunk;
    const int nk = min(kAttnChunk, pos0 + nt - k0);  // keys the block's last token sees
    // tokens of the block that see this chunk: tt >= tt0 (earlier positions end before k0)
    const int tt0 = max(0, k0 - pos0);
    const int R = (nt - tt0) * Gq;
    const long long page = page_table[j];
    const __nv_bfloat16* kp = kc + (page * nkv + g) * kPage * HD;
    const __nv_bfloat16* vp = vc + (page * nkv + g) * kPage * HD;
    // ---- loads, all in flight together: q rows -> shared (async); this warp's K fragments (keys
    // 16 ew + [0, 16), every k-step) and V fragments (its head dims, every key; zero past the last key)
    for (int i = et; i < R * (HD / 8); i += 128) {
        const int r = i / (HD / 8), part = i % (HD / 8);
        const int tt = tt0 + r / Gq, hq = g * Gq + r % Gq;
        cp_async16(S.q + r * kQStride + part * 8, a.qbuf + (static_cast<long long>(t0 + tt) * nh + hq) * HD + part * 8);
    }
    uint32_t kb[2][KS][2];
#pragma unroll
    for (int n8 = 0; n8 < 2; ++n8) {
        const uint32_t* kr = reinterpret_cast<const uint32_t*>(kp + static_cast<long long>(ew * 16 + n8 * 8 + gid) * HD);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            kb[n8][ks][0] = kr[ks * 8 + tig];
            kb[n8][ks][1] = kr[ks * 8 + 4 + tig];
        }
    }
    // V: column pair (base + 2 gid, + 1) of keys 16 ks + 2 tig + {0, 1, 8, 9}; n8 tile 2p holds the even
    // dims of the pair block, tile 2p + 1 the odd ones
    uint32_t vw[4][NP][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int pp = 0; pp < NP; ++pp)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int key = ks * 16 + 2 * tig + (e & 1) + (e >> 1) * 8;
                vw[ks][pp][e] = key < nk ? *reinterpret_cast<const uint32_t*>(
                                               vp + static_cast<long long>(key) * HD + ew * (HD / 4) + pp * 16 + 2 * gid)
                                         : 0u;
            }
    cp_async_wait_all();
    named_bar_sync(1, 128);
    if (et == 0) stamp(a, ph, 12);
    // ---- scores S = Q K^T for this warp's 16 keys, scaled and causally masked into shared memory
    {
        float sc[2][4] = {};
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const __nv_bfloat16* qa = S.q + gid * kQStride + ks * 16 + tig * 2;
            const uint32_t af[4] = {*reinterpret_cast<const uint32_t*>(qa),
                                    *reinterpret_cast<const uint32_t*>(qa + 8 * kQStride),
                                    *reinterpret_cast<const uint32_t*>(qa + 8),
                                    *reinterpret_cast<const uint32_t*>(qa + 8 * kQStride + 8)};
            mma16816(sc[0], af, kb[0][ks][0], kb[0][ks][1]);
            mma16816(sc[1], af, kb[1][ks][0], kb[1][ks][1]);
        }
        const float scale = rsqrtf(static_cast<float>(HD));
#pragma unroll
        for (int n8 = 0; n8 < 2; ++n8)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = gid + 8 * (i >> 1), key = ew * 16 + n8 * 8 + tig * 2 + (i & 1);
                const int tt = tt0 + row / Gq;
                const bool ok = row < R && key < nk && k0 + key <= pos0 + tt;
                S.p[row * kPStride + key] = ok ? sc[n8][i] * scale : -INFINITY;
            }
    }
    named_bar_sync(1, 128);
    if (et == 0) stamp(a, ph, 13);
    // ---- softmax of each row over the chunk's keys (warp ew takes rows ew, ew + 4, ...)
    for (int r = ew; r < R; r += 4) {
        float* pr = S.p + r * kPStride;
        const float s0 = pr[lane], s1 = pr[lane + 32];
        float mx = fmaxf(s0, s1);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const float e0 = s0 == -INFINITY ? 0.f : __expf(s0 - mx), e1 = s1 == -INFINITY ? 0.f : __expf(s1 - mx);
        float sum = e0 + e1;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        pr[lane] = e0;
        pr[lane + 32] = e1;
        if (lane == 0) {
            S.m[r] = mx;
            S.l[r] = sum;
        }
    }
    named_bar_sync(1, 128);
    if (et == 0) stamp(a, ph, 14);
    // ---- O = P V for this warp's head dims (P rounded to bf16 for the tensor cores; keys past a
    // row's limit carry p = 0 and zero V rows past the chunk's last key)
    float oc[NP][2][4] = {};
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const float* pa = S.p + gid * kPStride + ks * 16 + tig * 2;
        const float2 x0 = *reinterpret_cast<const float2*>(pa), x1 = *reinterpret_cast<const float2*>(pa + 8 * kPStride);
        const float2 x2 = *reinterpret_cast<const float2*>(pa + 8), x3 = *reinterpret_cast<const float2*>(pa + 8 * kPStride + 8);
        const uint32_t af[4] = {pack_bf16(x0.x, x0.y), pack_bf16(x1.x, x1.y), pack_bf16(x2.x, x2.y),
                                pack_bf16(x3.x, x3.y)};
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const uint32_t* w = vw[ks][pp];
            mma16816(oc[pp][0], af, __byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410));
            mma16816(oc[pp][1], af, __byte_perm(w[0], w[1], 0x7632), __byte_perm(w[2], w[3], 0x7632));
        }
    }
    // thread (gid, tig) holds dims base + 4 tig + [0, 4) of rows gid and gid + 8 for each pair block
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int row = gid + 8 * hr;
        if (row >= R) continue;
        const int tt = tt0 + row / Gq, hq = g * Gq + row % Gq, t = t0 + tt;
        const int nch = (pos0 + tt) / kAttnChunk + 1;
        const long long slot = (static_cast<long long>(t) * nh + hq) * a.max_chunks + j;
        const float inv_l = 1.0f / S.l[row];
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const int d = ew * (HD / 4) + pp * 16 + 4 * tig;
            const float4 o = make_float4(oc[pp][0][2 * hr], oc[pp][1][2 * hr], oc[pp][0][2 * hr + 1], oc[pp][1][2 * hr + 1]);
            if (nch == 1) {
                __nv_bfloat16* out = a.attn + static_cast<long long>(t) * a.q_dim + hq * HD + d;
                *reinterpret_cast<uint2*>(out) = make_uint2(pack_bf16(o.x * inv_l, o.y * inv_l), pack_bf16(o.z * inv_l, o.w * inv_l));
            } else {
                __stcg(reinterpret_cast<float4*>(a.part_o + slot * HD + d), o);
            }
        }
        if (nch > 1 && ew == 0 && tig == 0)
            __stcg(reinterpret_cast<float2*>(a.part_ml) + slot, make_float2(S.m[row], S.l[row]));
    }
}

struct BatchSmem {  // a batched forward's row -> lane map (the per-lane pointers stay in the
                   // __grid_constant__ kernel parameter, indexed in place)
    int n;
    int off[kMaxBatch + 1];
    int start[kMaxBatch], lc[kMaxBatch];
    int poff[kMaxBatch + 1];  // attention token blocks before lane b
};
// forward row t -> its lane (return) and position (*pos)
__device__ __forceinline__ int batch_row(const BatchSmem& B, int t, int* pos) {
    int b = 0;
    while (b + 1 < B.n && t >= B.off[b + 1]) ++b;
    *pos = B.start[b] + (t - B.off[b]);
    return b;
}

struct FwdSmem {
    uint64_t full[kFwdMaxStages], empty[kFwdMaxStages], tfull[2], tempty[2], drain;
    unsigned long long ep, tp_ep;
    uint32_t tslot;
    int sint[12];
    float rs[256];
    float red[128];
    float sval[128];
    int sidx[128];
    TpPeers peers;  // copy of FwdArgs::peers (dynamic indexing of kernel parameters would use local memory)
    BatchSmem bt;   // batched forward only
    union alignas(16) {
        float pre[16 * 128];  // GEMM phases: a finisher's presummed split-K partials, parked across the accumulator wait
        AttnSmem at;          // ATTN phases
    };
};
static_assert(sizeof(FwdSmem) <= kFwdMiscBytes, "misc shared state exceeds its budget");

// ATTN_COMBINE: one warp per (forward row t, q head): the position's chunk partials in chunk order
// (lane j holds chunk j's (max, sum); each lane HD/32 output dims; 8 chunks' loads per round trip).
template <int HD, bool kB>
__device__ __forceinline__ void attn_combine_phase(const FwdArgs& a, int start, int T, int gw, int GW, int lane,
                                                   const BatchSmem& B) {
    constexpr int DPL = HD / 32;
    const int nh = a.nh;
    for (int item = gw; item < T * nh; item += GW) {
        const int t = item / nh, hq = item % nh;
        int pos = start + t;
        if constexpr (kB) batch_row(B, t, &pos);
        const int nch = pos / kAttnChunk + 1;
        if (nch == 1) continue;  // written directly by the attention item
        const long long base = (static_cast<long long>(t) * nh + hq) * a.max_chunks;
        const float2* ml = reinterpret_cast<const float2*>(a.part_ml) + base;
        float M = -INFINITY;
        for (int jb = 0; jb < nch; jb += 32)
            if (jb + lane < nch) M = fmaxf(M, __ldcg(ml + jb + lane).x);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        float den = 0.f, acc[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = 0.f;
        for (int jb = 0; jb < nch; jb += 32) {
            const bool mine = jb + lane < nch;
            const float2 mv = mine ? __ldcg(ml + jb + lane) : make_float2(M, 0.f);
            const float wl = mine ? __expf(mv.x - M) : 0.f;
            const int n32 = min(32, nch - jb);
            for (int i0 = 0; i0 < n32; i0 += 8) {
                float v[8][DPL];
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int e = 0; e < DPL; ++e)
                        v[i][e] = i0 + i < n32 ? __ldcg(a.part_o + (base + jb + i0 + i) * HD + lane * DPL + e) : 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float wi = __shfl_sync(0xffffffffu, wl, (i0 + i) & 31);
                    const float li = __shfl_sync(0xffffffffu, mv.y, (i0 + i) & 31);
                    if (i0 + i < n32) {
                        den = fmaf(li, wi, den);
#pragma unroll
                        for (int e = 0; e < DPL; ++e) acc[e] = fmaf(v[i][e], wi, acc[e]);
                    }
                }
            }
        }
        const float inv = 1.0f / den;
        __nv_bfloat16* out = a.attn + static_cast<long long>(t) * a.q_dim + hq * HD + lane * DPL;
#pragma unroll
        for (int e = 0; e < DPL; e += 2)
            *reinterpret_cast<__nv_bfloat162*>(out + e) = __floats2bfloat162_rn(acc[e] * inv, acc[e + 1] * inv);
    }
}

// one attention phase of this CTA: items (token block, kv head, chunk) round-robin over the CTAs.  A
// token block is up to Tb = kAttnRows / G consecutive tokens of one sequence.
template <int HD, bool kB>
__device__ __forceinline__ void attn_phase(const FwdArgs& a, const FwdPhase& P, int start, int T, int c, int G,
                                           AttnSmem& S, const BatchSmem& B, int ph) {
    const int nkv = opaque(a.nkv), Tb = opaque(attn_block(a));
    int max_pos = start + T - 1;
    if constexpr (kB) {
        max_pos = 0;
        for (int b = 0; b < B.n; ++b) max_pos = max(max_pos, B.lc[b] - 1);
    }
    const int nch_max = max_pos / kAttnChunk + 1;
    int blocks = (T + Tb - 1) / Tb;
    if constexpr (kB) blocks = B.poff[B.n];
    const int items = blocks * nkv * nch_max;
    for (int item = c; item < items; item += G) {
        const int j = item % nch_max, rest = item / nch_max;
        const int g = rest % nkv, blk = rest / nkv;
        int t0, nt, pos0, b = 0;
        if constexpr (kB) {
            while (b + 1 < B.n && blk >= B.poff[b + 1]) ++b;
            t0 = B.off[b] + (blk - B.poff[b]) * Tb;
            nt = min(Tb, B.off[b + 1] - t0);
            pos0 = B.start[b] + (t0 - B.off[b]);
        } else {
            t0 = blk * Tb;
            nt = min(Tb, T - t0);
            pos0 = start + t0;
        }
        if (j * kAttnChunk > pos0 + nt - 1) continue;  // the chunk is in every block token's future
        const int32_t* pt = kB ? a.batch.page_table[b] : a.page_table;
        const __nv_bfloat16* kc = kB ? P.kc + a.batch.koff[b] : P.kc;
        const __nv_bfloat16* vc = kB ? P.vc + a.batch.voff[b] : P.vc;
        attn_item<HD>(a, S, g, j, t0, nt, pos0, pt, kc, vc, ph);
        named_bar_sync(1, 128);  // shared q / p are reused by the next item
        if (threadIdx.x == 64) stamp(a, ph, 15);
    }
}

// ------------------------------------------------------------------ GEMM tile finisher
// The last contributor of an output tile sums the split-K partials (fixed contributor order) and
// applies the fused epilogue.  This runs on the phase's critical path once per tile, with one warp
// per scheduler, so it is written for instruction-level parallelism: CH-column chunks (16 for decode
// forwards), loads issued before their uses, butterfly column reductions (31 shuffles per 32 lanes x
// CH columns) and compile-time loop bounds.
struct TileCtx {
    const FwdArgs* a;
    const FwdPhase* P;
    int p, m, n_contrib, my, first, tile_u0, U, A;
    uint32_t taddr;
    int tp, T, start, q, lane, et, r;
    float *rs, *red, *sval;
    int* sidx;
    unsigned long long tag;  // slot-flag value of this (forward, phase)
    unsigned long long xtag; // tensor-parallel exchange flag value of this (forward, phase)
    bool has_pre;            // pre holds the presummed partials of the other contributors (decode)
    float* pre;              // shared memory [16][128] (column-major: thread r reads pre[i*128 + r])
    const TpPeers* peers;    // tensor-parallel exchange buffers (shared-memory copy)
    const BatchSmem* bt;     // batched forward: rows -> lanes
    uint32_t tpre;           // TMEM columns (this warp's lanes) holding every chunk's presum (tp <= 64),
                             // valid when pre_all; else only chunk 0 lives in `pre`
    bool pre_all;
};

template <int CH>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[CH]) {
    if constexpr (CH == 16) tmem_ld16(taddr, v);
    else tmem_ld32(taddr, v);
}

// lane l ends with the sum over the warp's 32 lanes of column (l % CH)
template <int CH>
__device__ __forceinline__ float warp_colsum(float (&v)[CH], int lane) {
    if constexpr (CH == 16) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 16);
    }
#pragma unroll
    for (int s = CH / 2; s >= 1; s >>= 1) {
        const bool hi = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const float send = hi ? v[i] : v[i + s];
            const float keep = hi ? v[i + s] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
    return v[0];
}
// (max value, lowest index) — associative and commutative, so the same butterfly applies
__device__ __forceinline__ void amax_merge(float& bv, int& bi, float ov, int oi) {
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
}
template <int CH>
__device__ __forceinline__ void warp_colmax(float (&v)[CH], int (&id)[CH], int lane) {
    if constexpr (CH == 16) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            amax_merge(v[i], id[i], __shfl_xor_sync(0xffffffffu, v[i], 16), __shfl_xor_sync(0xffffffffu, id[i], 16));
    }
#pragma unroll
    for (int s = CH / 2; s >= 1; s >>= 1) {
        const bool hi = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const float sv = hi ? v[i] : v[i + s];
            const int si = hi ? id[i] : id[i + s];
            float kv = hi ? v[i + s] : v[i];
            int ki = hi ? id[i + s] : id[i];
            amax_merge(kv, ki, __shfl_xor_sync(0xffffffffu, sv, s), __shfl_xor_sync(0xffffffffu, si, s));
            v[i] = kv;
            id[i] = ki;
        }
    }
}

// Split tiles: the tile's first contributor (it processes the tile at the END of its range, the others
// at the START of theirs) is the designated finisher.  The others store their partial and release a
// per-slot flag; the finisher waits for the flags (usually long set) and sums the partials in
// contributor order — for decode forwards before its own accumulator is even ready.
__device__ __forceinline__ int slot_of(const TileCtx& x, int j) {  // partial slot of contributor first + j
    const int cj = x.first + j;
    return 2 * cj + (range_begin(cj, x.U, x.A) >= x.tile_u0 ? 0 : 1);
}
// one poller per contributor flag (all polls in flight together: a tile split over k CTAs costs one
// round trip, not k - 1), each acquiring its flag, then the epilogue barrier
__device__ __forceinline__ void wait_partials(const TileCtx& x) {
    for (int j = 1 + x.et; j < x.n_contrib; j += 128) {
        const unsigned long long* f = x.a->slot_flag + slot_of(x, j);
        Spin sp;
        while (ld_relaxed_u64(f) != x.tag)
            if (sp.tick(*x.a, 8, x.p)) break;
        fence_acq_rel_gpu();
    }
    named_bar_sync(1, 128);
}
// x.pre[i][r] = p_1 + p_2 + ... + p_{n-1} for columns [ch, ch + 16) of this thread's row, accumulated
// in shared memory (the thread's own row: no barrier) so no register array lives across the tail
__device__ __forceinline__ void presum(const TileCtx& x, int ch, const float* resid = nullptr) {
    const FwdArgs& a = *x.a;
    const int tp = x.tp, nc = min(16, tp - ch);
    float* pre = x.pre + x.r;
    for (int jb = 1; jb < x.n_contrib; jb += kBatch) {
        float xs[kBatch][16];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const bool load = jb + j < x.n_contrib;
            const float* Pj = a.ws + static_cast<long long>(load ? slot_of(x, jb + j) : 0) * tp * kBM + ch * kBM + x.r;
#pragma unroll
            for (int i = 0; i < 16; ++i) xs[j][i] = (load && i < nc) ? __ldcg(Pj + i * kBM) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float s2 = jb == 1 ? xs[0][i] : pre[i * kBM] + xs[0][i];
#pragma unroll
            for (int j = 1; j < kBatch; ++j)
                if (jb + j < x.n_contrib) s2 += xs[j][i];
            pre[i * kBM] = s2;
        }
    }
    if (resid) {  // a folded residual row: presum + resid, the one order on every path
#pragma unroll
        for (int i = 0; i < 16; ++i) pre[i * kBM] += i < nc ? __ldcg(resid + static_cast<long long>(i) * a.h) : 0.f;
    }
}

// the presum of chunk ch (+ the folded residual) added into v: from TMEM (every chunk presummed early),
// from `pre` (chunk 0 presummed early), or computed now
template <int CH>
__device__ __forceinline__ void add_presum(const TileCtx& x, int ch, const float* resid, float (&v)[CH]) {
    if (x.pre_all) {
#pragma unroll
        for (int k = 0; k < CH; k += 16) {
            float pv[16];
            tmem_ld16(x.tpre + ch + k, pv);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[k + i] += pv[i];
        }
        return;
    }
    if constexpr (CH == 16) {  // 32-column chunks only run with every presum in TMEM
        if (!x.has_pre || ch > 0) presum(x, ch, resid);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += x.pre[i * kBM + x.r];
    }
}
// early: every chunk's presum into TMEM (the accumulator is not ready yet; the partials are) — 32 columns
// at a time, two contributors' loads in flight, accumulated in registers in contributor order (the same
// order as presum: p_1 + p_2 + ... then + resid)
__device__ __forceinline__ void presum_all_to_tmem(const TileCtx& x, const float* resid0, long long resid_ld) {
    const FwdArgs& a = *x.a;
    const int tp = x.tp;
    for (int c0 = 0; c0 < ((a.dbg == 5 || a.dbg == 8) ? 16 : tp); c0 += 32) {
        const int ncol = min(32, tp - c0);
        float sacc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) sacc[i] = 0.f;
        for (int jb = 1; jb < x.n_contrib; jb += 2) {
            float xs[2][32];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const bool load = jb + j < x.n_contrib;
                const float* Pj = a.ws + static_cast<long long>(load ? slot_of(x, jb + j) : 0) * tp * kBM + c0 * kBM + x.r;
#pragma unroll
                for (int i = 0; i < 32; ++i) xs[j][i] = (load && i < ncol) ? __ldcg(Pj + i * kBM) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                sacc[i] = jb == 1 ? xs[0][i] : sacc[i] + xs[0][i];
                if (jb + 1 < x.n_contrib) sacc[i] += xs[1][i];
            }
        }
        if (resid0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) sacc[i] += i < ncol ? __ldcg(resid0 + static_cast<long long>(c0 + i) * resid_ld) : 0.f;
        }
        tmem_st16(x.tpre + c0, sacc);
        if (ncol > 16) tmem_st16(x.tpre + c0 + 16, sacc + 16);
    }
}

template <int CH, bool kTP, bool kB>
__device__ __forceinline__ void finish_tile(const TileCtx& x) {
    const FwdArgs& a = *x.a;
    const FwdPhase& P = *x.P;
    const int tp = x.tp, T = x.T, lane = x.lane, q = x.q, et = x.et, r = x.r, m = x.m;
    const int n = m * kBM + r;
    const int h = a.h;
    const bool tp_resid = kTP && P.epi == kFeResid;
    const int nth = h / kBM;
    if constexpr (kTP) if (tp_resid) {  // this rank's partial of tile m -> every rank's exchange slot [my rank][m]
        for (int ch = 0; ch < ((a.dbg == 5 || a.dbg == 7) ? 16 : tp); ch += CH) {
            float v[CH];
            tmem_ld<CH>(x.taddr + ch, v);
            const int nc = min(CH, tp - ch);
            if (x.n_contrib > 1) add_presum(x, ch, nullptr, v);
            for (int rr = 0; rr < a.tp_world; ++rr) {
                float* dst = x.peers->xch[rr] + (static_cast<long long>(a.tp_rank * nth + m) * 256 + ch) * kBM + r;
#pragma unroll
                for (int i = 0; i < CH; ++i)
                    if (i < nc) dst[i * kBM] = v[i];
            }
        }
        __threadfence_system();
        named_bar_sync(1, 128);
        // thread rr releases this rank's flag at rank rr and then waits for rank rr's flag here: all the
        // ranks' flags are polled in parallel (one round trip, not world - 1)
        if (et < a.tp_world) {
            st_release_sys_u64(x.peers->xflag[et] + a.tp_rank * nth + m, x.xtag);
            const unsigned long long* f = x.peers->xflag[a.tp_rank] + et * nth + m;
            Spin sp;
            while (ld_acquire_sys_u64(f) != x.xtag)
                if (sp.tick(a, 9, x.p)) break;
        }
        named_bar_sync(1, 128);
    }
    for (int ch = 0; ch < ((a.dbg == 5 || a.dbg == 7) ? 16 : tp); ch += CH) {
        float v[CH];
        const int nc = min(CH, tp - ch);
        if (kTP && tp_resid) {  // sum of the ranks' partials, rank order (identical on every rank)
            const float* src0 = x.peers->xch[a.tp_rank] + (static_cast<long long>(m) * 256 + ch) * kBM + r;
#pragma unroll
            for (int i = 0; i < CH; ++i) v[i] = i < nc ? __ldcg(src0 + i * kBM) : 0.f;
            for (int src = 1; src < a.tp_world; ++src) {
                const float* s1 = src0 + static_cast<long long>(src) * nth * 256 * kBM;
#pragma unroll
                for (int i = 0; i < CH; ++i) v[i] += i < nc ? __ldcg(s1 + i * kBM) : 0.f;
            }
        } else {
            tmem_ld<CH>(x.taddr + ch, v);
        }
        // own + (p_1 + p_2 + ...): fixed contributor order (per shape); a split residual tile adds the
        // residual to the presum (own + (presum + resid)) so the early finisher can do it before its
        // accumulator is ready — every path (row count, early or not) uses this one order
        const bool fold = !kTP && P.epi == kFeResid && x.n_contrib > 1;
        if (x.n_contrib > 1 && !tp_resid) add_presum(x, ch, fold ? a.resid + static_cast<long long>(ch) * h + n : nullptr, v);
        if (et == 0) stamp(a, x.p, 9);
        if (P.epi == kFeResid) {  // resid += acc; xb = bf16(resid); per-tile sum of squares
            float* o = a.resid + static_cast<long long>(ch) * h + n;
            float sq[CH];
#pragma unroll
            for (int i = 0; i < CH; ++i) sq[i] = (i < nc && !fold) ? __ldcg(o + static_cast<long long>(i) * h) : 0.f;
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                const float nv = fold ? v[i] : sq[i] + v[i];
                if (i < nc) {
                    o[static_cast<long long>(i) * h] = nv;
                    a.xb[static_cast<long long>(ch + i) * h + n] = __float2bfloat16_rn(nv);
                }
                sq[i] = i < nc ? nv * nv : 0.f;
            }
            if constexpr (CH == 32) {  // two 16-column halves: the CH = 16 summation order (batch invariance)
                float lo[16], hi[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    lo[i] = sq[i];
                    hi[i] = sq[16 + i];
                }
                x.red[q * 32 + lane] = warp_colsum<16>(lo, lane);
                x.sval[q * 32 + lane] = warp_colsum<16>(hi, lane);
                named_bar_sync(1, 128);
                if (et < 32 && ch + et < tp) {
                    const float* rb = et < 16 ? x.red : x.sval;
                    const int c = et & 15;
                    a.ssq[m * 256 + ch + et] = ((rb[c] + rb[32 + c]) + rb[64 + c]) + rb[96 + c];
                }
            } else {
                x.red[q * 32 + lane] = warp_colsum<CH>(sq, lane);
                named_bar_sync(1, 128);
                if (et < CH && ch + et < tp)
                    a.ssq[m * 256 + ch + et] = ((x.red[et] + x.red[32 + et]) + x.red[64 + et]) + x.red[96 + et];
            }
            named_bar_sync(1, 128);
        } else if (P.epi == kFeSilu) {  // rows interleaved 16 gate | 16 up per warp
            const int f = m * 64 + q * 16 + lane;
            __nv_bfloat16* o = a.act + static_cast<long long>(ch) * a.ffn_l + f;
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                const float g = v[i] * x.rs[ch + i];
                const float up = __shfl_down_sync(0xffffffffu, g, 16);
                if (lane < 16 && i < nc) o[static_cast<long long>(i) * a.ffn_l] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * up);
            }
        } else if (CH == 16 && P.epi == kFeQkv) {  // rstd scale, q/k RMSNorm, RoPE, q -> qbuf, k/v -> paged KV cache
            const int hd = a.hd, half = hd >> 1;
            const bool in_rows = n < P.n_out;  // warp-uniform (n_out % 64 == 0)
            const bool is_q = n < a.q_dim, is_k = !is_q && n < a.q_dim + a.kv_dim;
            const int base = is_q ? 0 : is_k ? a.q_dim : a.q_dim + a.kv_dim;
            const int head = (n - base) / hd, pr = (n - base) % hd, qh = pr >> 5;
            const int dd = lane < 16 ? 16 * qh + lane : half + 16 * qh + lane - 16;
            const __nv_bfloat16* nw = is_q ? P.qn : is_k ? P.kn : nullptr;
            const bool norm = in_rows && nw != nullptr;
            const float wd = norm ? __bfloat162float(nw[dd]) : 1.f;
            float xv[CH];
#pragma unroll
            for (int i = 0; i < CH; ++i) xv[i] = bf16r(v[i] * x.rs[ch + i]);
            {
                float sq[CH];
#pragma unroll
                for (int i = 0; i < CH; ++i) sq[i] = xv[i] * xv[i];
                x.red[q * 32 + lane] = warp_colsum<CH>(sq, lane);
            }
            named_bar_sync(1, 128);
            if (norm) {
                const int fq = q - qh, nwq = hd >> 5;
                const float inv_hd = 1.0f / static_cast<float>(hd);
                float ss[CH];
#pragma unroll
                for (int i = 0; i < CH; ++i) {
                    ss[i] = x.red[fq * 32 + i];
#pragma unroll
                    for (int w2 = 1; w2 < 4; ++w2)
                        if (w2 < nwq) ss[i] += x.red[(fq + w2) * 32 + i];
                }
#pragma unroll
                for (int i = 0; i < CH; ++i) xv[i] = bf16r(xv[i] * rsqrtf(ss[i] * inv_hd + a.eps) * wd);
            }
            named_bar_sync(1, 128);
            if (in_rows) {
                if (is_q || is_k) {  // RoPE: partner dim d +- hd/2 sits in lane ^ 16
                    const int dm = dd % half;
                    float2 cs[CH];
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        int pos = x.start + ch + i;
                        if constexpr (kB) if (ch + i < T) batch_row(*x.bt, ch + i, &pos);
                        cs[i] = ch + i < T ? __ldg(a.rope + static_cast<long long>(pos) * half + dm) : make_float2(1.f, 0.f);
                    }
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        const float partner = __shfl_xor_sync(0xffffffffu, xv[i], 16);
                        xv[i] = lane < 16 ? xv[i] * cs[i].x - partner * cs[i].y : xv[i] * cs[i].x + partner * cs[i].y;
                    }
                }
                if (is_q) {
                    __nv_bfloat16* dq = a.qbuf + (static_cast<long long>(ch) * a.nh + head) * hd + dd;
#pragma unroll
                    for (int i = 0; i < CH; ++i)
                        if (ch + i < T) dq[static_cast<long long>(i) * a.nh * hd] = __float2bfloat16_rn(xv[i]);
                } else if constexpr (kB) {  // each row appends to its own lane's cache
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        if (ch + i < T) {
                            int pos;
                            const int b = batch_row(*x.bt, ch + i, &pos);
                            __nv_bfloat16* kvc = is_k ? P.kc + a.batch.koff[b] : P.vc + a.batch.voff[b];
                            const int pg = __ldg(a.batch.page_table[b] + pos / kPage);
                            kvc[((static_cast<long long>(pg) * a.nkv + head) * kPage + pos % kPage) * hd + dd] =
                                __float2bfloat16_rn(xv[i]);
                        }
                    }
                } else {
                    __nv_bfloat16* kvc = is_k ? P.kc : P.vc;
                    int pg[CH];
#pragma unroll
                    for (int i = 0; i < CH; ++i) pg[i] = ch + i < T ? __ldg(a.page_table + (x.start + ch + i) / kPage) : 0;
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        const int pos = x.start + ch + i;
                        if (ch + i < T)
                            kvc[((static_cast<long long>(pg[i]) * a.nkv + head) * kPage + pos % kPage) * hd + dd] =
                                __float2bfloat16_rn(xv[i]);
                    }
                }
            }
        } else {  // kFeLogits: scaled logits; per-tile (max, lowest index) per column
            const bool ok = n < P.n_out;
#pragma unroll
            for (int i = 0; i < CH; ++i) v[i] *= x.rs[ch + i];
            if (a.logits && ok) {
#pragma unroll
                for (int i = 0; i < CH; ++i)
                    if (i < nc && ch + i < T) a.logits[static_cast<long long>(ch + i) * a.ld_logits + n] = v[i];
            }
            int id[CH];
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                id[i] = ok ? n + a.vocab_off : 0x7fffffff;
                if (!ok) v[i] = -INFINITY;
            }
            warp_colmax<CH>(v, id, lane);
            if (lane < CH) {
                x.sval[q * 32 + lane] = v[0];
                x.sidx[q * 32 + lane] = id[0];
            }
            named_bar_sync(1, 128);
            if (et < CH && et < nc) {
                float bv = x.sval[et];
                int bi = x.sidx[et];
                for (int qq = 1; qq < 4; ++qq) amax_merge(bv, bi, x.sval[qq * 32 + et], x.sidx[qq * 32 + et]);
                a.amax[static_cast<long long>(m) * tp + ch + et] = make_float2(bv, __int_as_float(bi));
            }
            named_bar_sync(1, 128);
        }
    }
}

// ------------------------------------------------------------------ the kernel
template <bool kTP, bool kB>  // TP exchange / batched lanes compiled in only where used (register pressure)
__global__ void __launch_bounds__(kFwdThreads, 2) fwd_kernel(const __grid_constant__ FwdArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ FwdSmem sm;  // static: the compiler keeps these in the shared address space (LDS/STS)
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = a.stages, tp = a.tp;
    const int bbytes = tp * kBK * 2;
    uint8_t* sA = smem;                   // stage s: weight tile at sA + s * 16 KiB
    uint8_t* sB = smem + S * kABytes;     //          activation rows at sB + s * tp * 128 B
    uint64_t* full = sm.full;  // one barrier per stage: weight tile + activation tile bytes
    uint64_t* empty = sm.empty;
    uint64_t* tfull = sm.tfull;
    uint64_t* tempty = sm.tempty;
    unsigned long long* sep = &sm.ep;
    uint32_t* tslot = &sm.tslot;
    int* sint = sm.sint;   // [0] start [1] T [2] L+c [3] flag
    float* rs = sm.rs;     // [256] rsqrt(mean square) per token column
    float* red = sm.red;   // [4][32]
    float* sval = sm.sval; // [4][32]
    int* sidx = sm.sidx;   // [4][32]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x, G = gridDim.x;
    // TMEM: nacc accumulators (+ one presum region when 16 < tp <= 64: two co-resident CTAs stay <= 512
    // columns; at tp = 16 the single chunk's presum stays in shared memory, measured faster for the draft)
    const bool tpre_on = a.tp > 16 && a.tp <= 64;
    const uint32_t tpre_col = static_cast<uint32_t>(a.nacc * a.acc_cols);
    const uint32_t ncols = [&] {
        const uint32_t used = tpre_col + (tpre_on ? static_cast<uint32_t>(a.acc_cols) : 0u);
        uint32_t n = 32;
        while (n < used) n <<= 1;
        return n;
    }();

    if (threadIdx.x == 0) {
        if constexpr (kB) {
            BatchSmem& B = sm.bt;
            B.n = a.batch.n;
            int off = 0, blocks = 0;
            const int Tb = attn_block(a);
            for (int b = 0; b < B.n; ++b) {
                const LaneState* Ls = a.batch.lane[b];
                const int st = min(Ls->kv_len, Ls->row0), lc = Ls->L + Ls->c;
                B.off[b] = off;
                B.start[b] = st;
                B.lc[b] = lc;
                B.poff[b] = blocks;
                off += lc - st;
                blocks += (lc - st + Tb - 1) / Tb;
            }
            B.off[B.n] = off;
            B.poff[B.n] = blocks;
            sint[0] = 0;
            sint[1] = off;
            sint[2] = 0;
        } else {
            const LaneState* L = a.lane;
            const int start = min(L->kv_len, L->row0), Lc = L->L + L->c;
            sint[0] = start;
            sint[1] = Lc - start;
            sint[2] = Lc;
        }
        *sep = *reinterpret_cast<volatile unsigned long long*>(a.epoch);
        g_wdtag = static_cast<int>(*sep & 0x3fffffffull) + 1;
        sm.tp_ep = a.tp_epoch ? *reinterpret_cast<volatile unsigned long long*>(a.tp_epoch) : *sep;
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128);
        }
        mbar_init(&sm.drain, 1);
        fence_barrier_init();
        if constexpr (kTP) sm.peers = a.peers;
    }
    if (warp == 1) tmem_alloc(tslot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int start = sint[0], T = sint[1];
    const unsigned long long ep = *sep;
    const unsigned long long tp_ep = sm.tp_ep;
    if (T < 1 || T > tp) {  // host contract violated: nothing consistent to compute
        if (c == 0 && threadIdx.x == 0) {
            if constexpr (kB) a.batch.lane[0]->error = 2;
            else a.lane->error = 2;
            atomicExch(a.err, 100);
        }
        __syncthreads();
        if (warp == 1) tmem_dealloc(tmem, ncols);
        return;
    }

    if (warp == 0) {
        if (lane == 0) {  // ======================================================== TMA producer
            // One ring of stages (weight tile + the unit's activation rows, one barrier).  Weight tiles are
            // issued as soon as a slot frees — across phase boundaries, never waiting on data; a stage's
            // barrier expects both byte counts, so the activation load can follow later (once the phase's
            // input is complete) and simply completes the transaction.  Only the T valid token rows are
            // loaded, in as few copies as possible (the producer's issue rate bounds the stream): one box of
            // 4 / 8 / 16 rows up to 16 tokens, else 64-row boxes + one 32 and / or one 16 (tp is a multiple of
            // 16, so every box lands inside the stage).  Rows >= T keep stale data that reaches only padded
            // columns.
            for (int i = 0; i < 5; ++i) tma_prefetch_desc(&a.wmaps[i]);
            // DBL_FWD_DBG=1 (timing experiment, results invalid): load 16 activation rows whatever T is
            const int Tx = a.dbg == 1 ? min(T, 16) : T;
            const int n16 = (Tx + 15) / 16;
            const int xb_i = Tx <= 4 ? 0 : Tx <= 8 ? 1 : 2;  // single box (T <= 16): 4 << xb_i rows
            const int x_rows_total = Tx <= 16 ? (4 << xb_i) : n16 * 16;
            const uint32_t stage_tx = static_cast<uint32_t>(kABytes + x_rows_total * kBK * 2);
            for (int i = 0; i < 3; ++i)
                for (int b = 0; b < 5; ++b) tma_prefetch_desc(&a.xmaps[i][b]);
            Cur w{}, x{};
            seek(w, a, c, G);
            seek(x, a, c, G);
            Ring wr, xr;
            auto issue_x = [&]() {  // the activation rows of unit x into stage xr
                uint8_t* dst = sB + xr.st * bbytes;
                const CUtensorMap* xm = a.xmaps[x.xmap];
                if (Tx <= 16) {
                    tma_load_2d(dst, &xm[xb_i], &full[xr.st], x.kb * kBK, 0, kEvictLast);
                } else {
                    const int q64 = n16 >> 2, rem = n16 & 3;
                    for (int j = 0; j < q64; ++j)
                        tma_load_2d(dst + j * 64 * kBK * 2, &xm[4], &full[xr.st], x.kb * kBK, j * 64, kEvictLast);
                    int row = q64 * 64;
                    if (rem & 2) {
                        tma_load_2d(dst + row * kBK * 2, &xm[3], &full[xr.st], x.kb * kBK, row, kEvictLast);
                        row += 32;
                    }
                    if (rem & 1) tma_load_2d(dst + row * kBK * 2, &xm[2], &full[xr.st], x.kb * kBK, row, kEvictLast);
                }
            };
            int pending = 0;  // units whose weights are issued but whose activations are not
            int n_fill = 0;   // stages issued (watchdog abort: the copies to wait for)
            int dep_phase = -1, stamped = -1;
            Spin spin;
            while (w.p < a.n_ph || pending > 0) {
                bool prog = false;
                if (w.p < a.n_ph && mbar_test(&empty[wr.st], wr.ph ^ 1u)) {
                    if (stamped != w.p) {
                        stamp(a, w.p, 0);
                        stamped = w.p;
                    }
                    mbar_arrive_expect_tx(&full[wr.st], stage_tx);
                    // tiled weight image: tile (row block, kb) is rows [(blk * KB + kb) * 128, +128) of 128 B
                    tma_load_2d(sA + wr.st * kABytes, &a.wmaps[w.wmap], &full[wr.st], 0,
                                ((w.wrow / kBM + w.m) * w.KB + w.kb) * kBM,
                                kEvictFirst);
                    ++n_fill;
                    wr.next(S);
                    ++pending;
                    step(w, a, c, G);
                    prog = true;
                }
                if (pending > 0) {  // activations: only once the phase's input is complete
                    bool ok = x.p == dep_phase;
                    if (!ok && dep_ok(a, x.dep, ep)) {
                        fence_proxy_async_global();
                        dep_phase = x.p;
                        ok = true;
                        stamp(a, x.p, 1);
                    }
                    if (ok) {
                        issue_x();
                        xr.next(S);
                        --pending;
                        step(x, a, c, G);
                        prog = true;
                    }
                }
                if (prog) {
                    spin = Spin{};
                } else {
                    // Nothing issuable: park on the next ring slot (the hardware wakes the thread when it
                    // frees).  While activations wait on a dependency, bound the park so the flag is
                    // polled again within ~0.25 us.
                    if (spin.tick(a, 1, pending > 0 ? x.p : w.p)) {
                        // abort: complete every issued stage's transaction (the pending units' activation
                        // rows, stale) and wait until all issued copies have landed before exiting
                        for (; pending > 0; --pending) {
                            issue_x();
                            xr.next(S);
                            step(x, a, c, G);
                        }
                        for (int i = 0; i < S && i < n_fill; ++i)
                            while (!mbar_try(&full[i], static_cast<uint32_t>(((n_fill - 1 - i) / S) & 1))) {
                            }
                        break;
                    }
                    if (w.p < a.n_ph) {
                        if (pending > 0) mbar_try_hint(&empty[wr.st], wr.ph ^ 1u, 250);
                        else mbar_try(&empty[wr.st], wr.ph ^ 1u);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ========================================================== MMA issuer
            const uint32_t idesc = idesc_bf16_m128(tp);
            Cur k{};
            seek(k, a, c, G);
            Ring rr, tr;  // stage ring; TMEM accumulator ring (nacc buffers)
            int mma_stamped = -1;
            bool abort = false;
            while (k.p < a.n_ph && !abort) {
                const int p = k.p;
                const int n = min(k.e - k.u, k.KB - k.kb);  // units of this tile in this CTA's range
                abort = mbar_wait_wd(&tempty[tr.st], tr.ph ^ 1u, a, 2, p);
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(tr.st * a.acc_cols);
                for (int i = 0; i < n && !abort; ++i) {
                    if (mbar_wait_wd(&full[rr.st], rr.ph, a, 3, p)) {
                        abort = true;
                        break;
                    }
                    tc_fence_after();
                    if (p != mma_stamped) {
                        stamp(a, p, 4);  // first MMA of the phase
                        mma_stamped = p;
                    }
                    const uint64_t ad = umma_desc_sw128(smem_u32(sA + rr.st * kABytes));
                    const uint64_t bd = umma_desc_sw128(smem_u32(sB + rr.st * bbytes));
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        mma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
                    mma_commit(&empty[rr.st]);
                    rr.next(S);
                    step(k, a, c, G);
                }
                if (abort) break;
                mma_commit(&tfull[tr.st]);
                tr.next(a.nacc);
                stamp(a, p, 5);  // last MMA issued (so far) for the phase
            }
            if (abort) {  // the issued MMAs retire before the accumulator memory is released
                mma_commit(&sm.drain);
                while (!mbar_try(&sm.drain, 0u)) {
                }
            }
        }
    } else {  // ============================================ epilogue + aux work (128 threads)
        const int q = warp & 3;            // TMEM lane quadrant of this warp
        const int r = q * 32 + lane;       // tile row
        const int et = threadIdx.x - 64;   // 0..127
        const int ew = et >> 5;            // aux warp index 0..3
        const int gw = c * 4 + ew, GW = G * 4;
        const int h = a.h;
        int it = 0;
        auto signal = [&](int p) {  // this CTA's contribution to phase p is written
            fence_proxy_async_global();
            named_bar_sync(1, 128);
            if (et == 0) {
                red_release_add_u64(a.done + p, 1ull);
                stamp(a, p, 2);  // last contribution signalled
            }
        };
        auto acquire = [&](int p) {
            if (et == 0) wait_dep(a, p, ep, 5);
            named_bar_sync(1, 128);
        };
        if constexpr (!kB) {  // warm L2: this forward's embedding rows and RoPE rows (tiny, cold, on the critical path)
            const int gt = c * 128 + et, GT = G * 128;
            for (int t = gt; t < T; t += GT) {
                const int tok = a.buf[start + t];
                l2_warm(a.embed + static_cast<long long>(valid_token(tok, a) ? tok : 0) * h, h * 2, 0, 1);
            }
            if (gt == GT - 1) l2_warm(a.rope + static_cast<long long>(start) * (a.hd / 2), T * (a.hd / 2) * 8LL, 0, 1);
        }
        for (int p = 0; p < a.n_ph; ++p) {
            const FwdPhase& P = a.ph[p];
            if (!kB && P.kind == kPhGemm && P.epi == kFeQkv) {
                // warm L2 with this layer's norm weights and the context's K/V (read by ATTN next)
                const int pages = (start + T + kPage - 1) / kPage;
                const long long kv_bytes = static_cast<long long>(pages) * a.nkv * kPage * a.hd * 2;
                if (et < 2) l2_warm(P.kc, kv_bytes, c * 2 + et, G * 2);
                else if (et < 4) l2_warm(P.vc, kv_bytes, c * 2 + et - 2, G * 2);
                else if (et == 4 && c == 0 && P.qn) l2_warm(P.qn, a.hd * 2, 0, 1);
                else if (et == 5 && c == 0 && P.kn) l2_warm(P.kn, a.hd * 2, 0, 1);
            }
            if (P.kind == kPhEmbed) {  // ------------------------------------------- embedding
                const int nt = h / kBM;
                const int items = tp * nt;
                for (int item = gw; item < items; item += GW) {
                    const int t = item / nt, mt = item % nt;
                    int tok = 0;
                    if (t < T) {
                        if constexpr (kB) {
                            int pos;
                            const int b = batch_row(sm.bt, t, &pos);
                            tok = a.batch.buf[b][pos];
                        } else {
                            tok = a.buf[start + t];
                        }
                    }
                    if (!valid_token(tok, a)) tok = 0;  // ids outside the vocab (a draft's or a datastore's) are
                                                        // never accepted; their rows only need to be safe
                    const int col = mt * kBM + lane * 4;
                    const uint2 raw = *reinterpret_cast<const uint2*>(a.embed + static_cast<long long>(tok) * h + col);
                    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
                    const float2 f0 = __bfloat1622float2(b2[0]), f1 = __bfloat1622float2(b2[1]);
                    *reinterpret_cast<float4*>(a.resid + static_cast<long long>(t) * h + col) =
                        make_float4(f0.x, f0.y, f1.x, f1.y);
                    *reinterpret_cast<uint2*>(a.xb + static_cast<long long>(t) * h + col) = raw;
                    float ss = fmaf(f0.x, f0.x, 0.f);
                    ss = fmaf(f0.y, f0.y, ss);
                    ss = fmaf(f1.x, f1.x, ss);
                    ss = fmaf(f1.y, f1.y, ss);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
                    if (lane == 0) a.ssq[mt * 256 + t] = ss;
                }
                signal(p);
            } else if (P.kind == kPhGemm) {  // ------------------------------------- GEMM tiles
                const Range rg = cta_range(P, c, G);
                if (rg.b0 >= rg.b1) continue;
                acquire(P.dep);
                stamp(a, p, 3);
                if (P.epi != kFeResid) {  // column scale of the folded RMSNorm
                    const int nt = h / kBM;
                    for (int t = et; t < tp; t += 128) {
                        float s = 0.f;
                        for (int m = 0; m < nt; ++m) s += __ldcg(a.ssq + m * 256 + t);
                        rs[t] = rsqrtf(s * (1.0f / static_cast<float>(h)) + a.eps);
                    }
                    named_bar_sync(1, 128);
                }
                const int U = P.units, A = P.active;
                const unsigned long long tag = (ep << 12) | static_cast<unsigned long long>(p + 1);
                for (int u = rg.b0; u < rg.b1;) {
                    const int m = u / P.kb;
                    const int tile_u0 = m * P.kb, tile_u1 = tile_u0 + P.kb;
                    const int stop = min(tile_u1, rg.b1);
                    const int first = owner_of(tile_u0, U, A), last = owner_of(tile_u1 - 1, U, A);
                    const int n_contrib = static_cast<int>(last - first + 1);
                    const int my = static_cast<int>(rg.ci - first);
                    const int buf = it % a.nacc;
                    const uint32_t taddr = tmem + static_cast<uint32_t>(buf * a.acc_cols) + (static_cast<uint32_t>(q * 32) << 16);
                    const bool finisher = my == 0;
                    TileCtx tc{&a, &P, p, m, n_contrib, my, first, tile_u0, U, A, taddr, tp, T, start,
                               q, lane, et, r, rs, red, sval, sidx, tag, (tp_ep << 12) | static_cast<unsigned long long>(p + 1),
                               false, sm.pre, &sm.peers, &sm.bt,
                               tmem + tpre_col + (static_cast<uint32_t>(q * 32) << 16), false};
                    const bool early = finisher && n_contrib > 1;
                    if (early) {  // the other contributors are (nearly always) done: sum them now, the
                                  // residual folded in too (off the tail's chain) — every chunk into TMEM
                                  // (tp <= 64), else the first chunk into sm.pre
                        wait_partials(tc);
                        const float* rz = !kTP && P.epi == kFeResid ? a.resid + m * kBM + r : nullptr;
                        if (tpre_on) {
                            presum_all_to_tmem(tc, rz, h);
                            tc.pre_all = true;
                        } else {
                            presum(tc, 0, rz);
                            tc.has_pre = true;
                        }
                    }
                    mbar_wait_wd(&tfull[buf], static_cast<uint32_t>((it / a.nacc) & 1), a, 6, p);
                    tc_fence_after();
                    if (et == 0) stamp(a, p, 7);  // accumulator of this CTA's latest tile ready
                    if (!finisher) {  // partial -> slot, then release the slot flag
                        const int slot = 2 * rg.ci + (u == rg.b0 ? 0 : 1);
                        float* Pp = a.ws + static_cast<long long>(slot) * tp * kBM;
                        for (int ch = 0; ch < ((a.dbg == 5 || a.dbg == 6) ? 16 : tp); ch += 16) {
                            float v[16];
                            tmem_ld16(taddr + ch, v);
#pragma unroll
                            for (int i = 0; i < 16; ++i) __stcg(Pp + (ch + i) * kBM + r, v[i]);
                        }
                        named_bar_sync(1, 128);
                        if (et == 0) st_release_u64(a.slot_flag + slot, tag);
                    } else {
                        if (et == 0) stamp(a, p, 8);
                        if (n_contrib > 1 && !early) wait_partials(tc);
                        // 32-column chunks for 16 < tp <= 64 (every presum is in TMEM) outside QKV (its RoPE /
                        // head-norm epilogue keeps 16), else 16-column chunks
                        if constexpr (!kTP) {  // (the exchange path keeps 16: 32 would spill there)
                            if (tp > 16 && tp <= 64 && P.epi != kFeQkv) finish_tile<32, kTP, kB>(tc);
                            else finish_tile<16, kTP, kB>(tc);
                        } else {
                            finish_tile<16, kTP, kB>(tc);
                        }
                    }
                    if (et == 0 && finisher) stamp(a, p, 10);
                    tc_fence_before();
                    mbar_arrive(&tempty[buf]);
                    ++it;
                    if (finisher) signal(p);
                    if (et == 0 && finisher) stamp(a, p, 11);
                    u = stop;
                }
                if (et == 0) stamp(a, p, 6);  // this CTA's tiles of the phase are done
            } else if (P.kind == kPhAttn) {  // ------------------------- split-KV causal attention
                acquire(P.dep);
                stamp(a, p, 3);
                if (a.hd == 128) attn_phase<128, kB>(a, P, start, T, c, G, sm.at, sm.bt, p);
                else attn_phase<64, kB>(a, P, start, T, c, G, sm.at, sm.bt, p);
                if (lane == 0) stamp(a, p, 8 + ew);  // each aux warp's last item done
                signal(p);
            } else if (P.kind == kPhCombine) {  // --------------- split-KV partials -> attention output
                acquire(P.dep);
                if (a.hd == 128) attn_combine_phase<128, kB>(a, start, T, gw, GW, lane, sm.bt);
                else attn_combine_phase<64, kB>(a, start, T, gw, GW, lane, sm.bt);
                signal(p);
            } else {  // kPhArgmax ----------------------------------------- final argmax + cursor
                acquire(P.dep);
                const int n_tiles = a.ph[P.dep].n_tiles;
                for (int t = gw; t < T; t += GW) {
                    float bv = -INFINITY;
                    int bi = 0x7fffffff;
                    for (int m = lane; m < n_tiles; m += 32) {
                        const float2 pr2 = __ldcg(a.amax + static_cast<long long>(m) * tp + t);
                        const int pi = __float_as_int(pr2.y);
                        if (pr2.x > bv || (pr2.x == bv && pi < bi)) { bv = pr2.x; bi = pi; }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                    }
                    if (lane == 0) {
                        if constexpr (kB) {
                            int pos;
                            const int b = batch_row(sm.bt, t, &pos);
                            a.batch.argmax[b][pos] = (bi == 0x7fffffff || bv != bv || aborted(a)) ? -1 : bi;
                        } else if constexpr (!kTP) {
                            a.argmax[start + t] = (bi == 0x7fffffff || bv != bv || aborted(a)) ? -1 : bi;
                        } else {  // this rank's shard winner -> every rank's exchange slot [my rank][t]
                            for (int rr = 0; rr < a.tp_world; ++rr)
                                sm.peers.axch[rr][a.tp_rank * 256 + t] = make_float2(bv, __int_as_float(bi));
                        }
                    }
                }
                if constexpr (kTP) __threadfence_system();
                signal(p);
                if (c == 0 && et == 0) {  // the forward is complete once every CTA has signalled
                    wait_dep(a, p, ep, 7);
                    if constexpr (kTP) {  // vocab-parallel argmax: (max, lowest global id) over ranks
                        const unsigned long long tag = (tp_ep << 12) | static_cast<unsigned long long>(p + 1);
                        __threadfence_system();
                        for (int rr = 0; rr < a.tp_world; ++rr) st_release_sys_u64(sm.peers.aflag[rr] + a.tp_rank, tag);
                        for (int src = 0; src < a.tp_world; ++src) {
                            Spin sp;
                            while (ld_acquire_sys_u64(sm.peers.aflag[a.tp_rank] + src) != tag)
                                if (sp.tick(a, 10, p)) break;
                        }
                        for (int t = 0; t < T; ++t) {
                            float bv = -INFINITY;
                            int bi = 0x7fffffff;
                            for (int src = 0; src < a.tp_world; ++src) {
                                const float2 w = __ldcg(sm.peers.axch[a.tp_rank] + src * 256 + t);
                                const int wi = __float_as_int(w.y);
                                if (w.x > bv || (w.x == bv && wi < bi)) { bv = w.x; bi = wi; }
                            }
                            a.argmax[start + t] = (bi == 0x7fffffff || bv != bv || aborted(a)) ? -1 : bi;
                        }
                    }
                    if constexpr (kB) {
                        for (int b = 0; b < sm.bt.n; ++b) {
                            a.batch.lane[b]->start = sm.bt.start[b];
                            a.batch.lane[b]->kv_len = sm.bt.lc[b];
                            if (a.batch.row_base) a.batch.row_base[b] = sm.bt.off[b] - sm.bt.start[b];
                        }
                    } else {
                        a.lane->start = start;
                        a.lane->kv_len = sint[2];
                    }
                    __threadfence();
                    *reinterpret_cast<volatile unsigned long long*>(a.epoch) = ep + 1;
                    if (a.tp_epoch) *reinterpret_cast<volatile unsigned long long*>(a.tp_epoch) = tp_ep + 1;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, ncols);
    }
}

}  // namespace

void fwd_prepare() {
    static std::once_flag once;
    std::call_once(once, [] {
        CUDA_CHECK(cudaFuncSetAttribute(fwd_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024 - kFwdMiscBytes));
        CUDA_CHECK(cudaFuncSetAttribute(fwd_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024 - kFwdMiscBytes));
        CUDA_CHECK(cudaFuncSetAttribute(fwd_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024 - kFwdMiscBytes));
        // the whole unified L1 as shared memory: a target CTA (~140 KB) and a draft CTA (~68 KB) must
        // co-reside on every SM whichever launches first (the driver would otherwise size the carveout
        // for the first kernel alone and the second persistent grid would wait for the first to finish)
        for (auto k : {fwd_kernel<false, false>, fwd_kernel<true, false>, fwd_kernel<false, true>})
            CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared));
    });
}

int fwd_smem_budget(int budget) {  // DBL_FWD_SMEM_KB overrides (A/B)
    static const int kb = [] {
        const char* e = std::getenv("DBL_FWD_SMEM_KB");
        return e ? std::atoi(e) : 0;
    }();
    return kb > 0 ? std::min(kb, 227) * 1024 : budget;
}

int fwd_stages(int tp, int budget, size_t* smem) {
    const int stage = kABytes + tp * kBK * 2;
    // kFwdMiscBytes: the static FwdSmem.  At least two stages even past the budget (a wide batched
    // forward in the draft role then does not co-reside with the target: the launches serialize)
    const int s = std::max(2, (fwd_smem_budget(budget) - 1024 - kFwdMiscBytes) / stage);
    if (1024 + kFwdMiscBytes + 2 * stage > 227 * 1024)
        throw_invalid("stream forward: token bucket too large for the shared-memory ring");
    const int stages = std::min(s, kFwdMaxStages);
    *smem = 1024 + static_cast<size_t>(stages) * stage;
    return stages;
}

namespace {
struct FwdTrace {
    DevBuf<unsigned long long> buf;
    int n_ph = 0, grid = 0;
};
FwdTrace& fwd_trace() {
    static FwdTrace t;
    return t;
}
}  // namespace

unsigned long long* fwd_trace_buffer(int n_ph, int grid) {
    static const bool on = [] {
        const char* e = std::getenv("DBL_FWD_TRACE");
        return e && e[0] == '1';
    }();
    if (!on) return nullptr;
    FwdTrace& t = fwd_trace();
    const size_t need = static_cast<size_t>(n_ph) * grid * 16;
    if (t.buf.n < need) {
        t.buf.alloc(need);
        t.buf.zero();
    }
    t.n_ph = n_ph;
    t.grid = grid;
    return t.buf.p;
}

void fwd_trace_read(unsigned long long* dst, long long cap, int* n_ph, int* grid) {
    FwdTrace& t = fwd_trace();
    *n_ph = t.n_ph;
    *grid = t.grid;
    const long long need = static_cast<long long>(t.n_ph) * t.grid * 16;
    if (need == 0) return;
    if (cap < need) throw_invalid("trace buffer too small");
    CUDA_CHECK(cudaDeviceSynchronize());
    CUDA_CHECK(cudaMemcpy(dst, t.buf.p, need * 8, cudaMemcpyDeviceToHost));
}

void fwd_launch(const FwdArgs& a, int grid, size_t smem, cudaStream_t s, bool coop_in) {
    // Cooperative launch: the forward's CTAs wait on each other (phase counters), so they must be
    // co-resident — gang scheduling guarantees it even when a draft forward or another shard's
    // forward shares the GPU (a partially resident persistent grid could otherwise spin forever).
    fwd_prepare();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFwdThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    static const bool coop_env = [] {  // DBL_FWD_COOP=0: plain launches (experiment)
        const char* e = std::getenv("DBL_FWD_COOP");
        return !(e && e[0] == '0');
    }();
    cfg.numAttrs = coop_env && coop_in ? 1 : 0;
    if (a.batch.n > 0) {
        if (a.tp_world > 1) throw_invalid("batched forward: tensor-parallel lanes are not supported");
        CUDA_CHECK(cudaLaunchKernelEx(&cfg, fwd_kernel<false, true>, a));
    } else if (a.tp_world > 1) {
        CUDA_CHECK(cudaLaunchKernelEx(&cfg, fwd_kernel<true, false>, a));
    } else {
        CUDA_CHECK(cudaLaunchKernelEx(&cfg, fwd_kernel<false, false>, a));
    }
    ++launch_counter();
}

}  // namespace dbl
