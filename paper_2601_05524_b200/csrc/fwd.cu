// The persistent stream-forward kernel (design: fwd.cuh).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "fwd.cuh"
#include "sm100.cuh"
#include "tf_kernels.cuh"

namespace dbl {

namespace {

using namespace sm100;

constexpr int kBM = 128, kBK = 64;
constexpr int kABytes = kBM * kBK * 2;  // one 128 x 64 bf16 weight tile
constexpr unsigned long long kWatchdogNs = 4000000000ull;
constexpr int kBatch = 4;               // split-K partials: 4 contributors x 16 columns of loads in flight

// ------------------------------------------------------------------ small helpers
__device__ __noinline__ void watchdog_fire(int* err, int code, int phase) {
    atomicExch(err, code);
    printf("dbl fwd_kernel watchdog: CTA %d thread %d stuck (role %d, phase %d)\n", blockIdx.x, threadIdx.x, code,
           phase);
    __trap();
}
struct Spin {
    unsigned long long t0 = 0;
    unsigned n = 0;
    __device__ __forceinline__ void tick(int* err, int code, int phase) {
        if ((++n & 127u) == 0) {
            const unsigned long long t = globaltimer();
            if (!t0) t0 = t;
            else if (t - t0 > kWatchdogNs) watchdog_fire(err, code, phase);
        }
    }
};
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t par, int* err, int code, int phase) {
    Spin s;
    while (!mbar_try(bar, par)) s.tick(err, code, phase);
}

// A phase's stream-K split: phase-local CTA ci takes units [ci*U/A, (ci+1)*U/A).  Unit counts fit in
// 32 bits (host-checked); products are formed in 64 bits once per phase, never in the per-tile loops.
struct Range {
    int b0, b1;
    int ci;  // phase-local CTA index
};
__device__ __forceinline__ int range_begin(int ci, int U, int A) {
    return static_cast<int>(static_cast<long long>(ci) * U / A);
}
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
__device__ __forceinline__ int owner_of(int u, int U, int A) {
    return static_cast<int>(((static_cast<long long>(u) + 1) * A - 1) / U);
}

__device__ __forceinline__ bool dep_ok(const FwdArgs& a, int p, unsigned long long ep) {
    if (p < 0) return true;
    if (ld_relaxed_u64(a.done + p) < (ep + 1) * static_cast<unsigned long long>(a.ph[p].count)) return false;
    fence_acq_rel_gpu();
    return true;
}
__device__ __forceinline__ void wait_dep(const FwdArgs& a, int p, unsigned long long ep, int code) {
    Spin s;
    while (!dep_ok(a, p, ep)) s.tick(a.err, code, p);  // each probe is an L2 round trip
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

// One (token, q head, 64-key chunk) of split-KV causal attention, one warp.  Scores: lane = key
// (all of the key row's loads in flight at once); P*V: lane = HD/32 contiguous dims.  Chunks of a
// position combine in chunk order (the last-arriving warp does it), so the result depends on the
// position only — never on how many tokens the forward carries.
template <int HD>
__device__ __forceinline__ void attn_item(const FwdArgs& a, const FwdPhase& P, int t, int hq, int j, int start,
                                          float* q_s, float* p_s, int lane) {
    constexpr int DPL = HD / 32;
    const int nh = a.nh, kvh = hq / (nh / a.nkv);
    const int pos = start + t, k0 = j * kAttnChunk;
    const int nch = pos / kAttnChunk + 1, nk = min(kAttnChunk, pos - k0 + 1);
    const long long page = a.page_table[j];
    const __nv_bfloat16* kp = P.kc + (page * a.nkv + kvh) * kPage * HD;
    const __nv_bfloat16* vp = P.vc + (page * a.nkv + kvh) * kPage * HD;
    const __nv_bfloat16* qs = a.qbuf + (static_cast<long long>(t) * nh + hq) * HD;
#pragma unroll
    for (int e = 0; e < DPL; ++e) q_s[lane * DPL + e] = __bfloat162float(qs[lane * DPL + e]);
    __syncwarp();
    const float scale = rsqrtf(static_cast<float>(HD));
    float sc[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        const int kk = lane + 32 * h2;
        sc[h2] = -INFINITY;
        if (kk < nk) {
            const uint4* kr = reinterpret_cast<const uint4*>(kp + static_cast<long long>(kk) * HD);
            uint4 w[HD / 8];
#pragma unroll
            for (int d8 = 0; d8 < HD / 8; ++d8) w[d8] = kr[d8];
            float acc = 0.f;
#pragma unroll
            for (int d8 = 0; d8 < HD / 8; ++d8) {
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&w[d8]);
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    const float2 kf = __bfloat1622float2(b2[e2]);
                    acc = fmaf(q_s[d8 * 8 + 2 * e2], kf.x, acc);
                    acc = fmaf(q_s[d8 * 8 + 2 * e2 + 1], kf.y, acc);
                }
            }
            sc[h2] = acc * scale;
        }
    }
    float mx = fmaxf(sc[0], sc[1]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float e0 = lane < nk ? __expf(sc[0] - mx) : 0.f, e1 = lane + 32 < nk ? __expf(sc[1] - mx) : 0.f;
    p_s[lane] = e0;
    p_s[lane + 32] = e1;
    float l = e0 + e1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    __syncwarp();
    float o[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[e] = 0.f;
    const __nv_bfloat16* vl = vp + lane * DPL;
#pragma unroll 8
    for (int i = 0; i < nk; ++i) {
        const float pi = p_s[i];
        if constexpr (DPL == 4) {
            const uint2 raw = *reinterpret_cast<const uint2*>(vl + static_cast<long long>(i) * HD);
            const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
            const float2 v0 = __bfloat1622float2(b2[0]), v1 = __bfloat1622float2(b2[1]);
            o[0] = fmaf(pi, v0.x, o[0]);
            o[1] = fmaf(pi, v0.y, o[1]);
            o[2] = fmaf(pi, v1.x, o[2]);
            o[3] = fmaf(pi, v1.y, o[3]);
        } else {
            const float2 v0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vl + static_cast<long long>(i) * HD));
            o[0] = fmaf(pi, v0.x, o[0]);
            o[1] = fmaf(pi, v0.y, o[1]);
        }
    }
    __nv_bfloat16* out = a.attn + static_cast<long long>(t) * a.q_dim + hq * HD + lane * DPL;
    if (nch == 1) {
        const float inv = 1.0f / l;
#pragma unroll
        for (int e = 0; e < DPL; ++e) out[e] = __float2bfloat16_rn(o[e] * inv);
        return;
    }
    const long long slot = (static_cast<long long>(t) * nh + hq) * a.max_chunks + j;
#pragma unroll
    for (int e = 0; e < DPL; ++e) __stcg(a.part_o + slot * HD + lane * DPL + e, o[e]);
    if (lane == 0) {
        __stcg(a.part_ml + 2 * slot, mx);
        __stcg(a.part_ml + 2 * slot + 1, l);
    }
    __syncwarp();
    int last_in = 0;
    if (lane == 0) {  // one acq_rel RMW (the warp's stores are ordered before it by __syncwarp)
        int* cnt = a.attn_cnt + t * nh + hq;
        last_in = atom_add_acq_rel_gpu(cnt, 1) == nch - 1;
        if (last_in) *cnt = 0;
    }
    last_in = __shfl_sync(0xffffffffu, last_in, 0);
    if (!last_in) return;
    __syncwarp();  // lane 0's acquire orders the other lanes' reads of the partials
    // combine this position's chunks in chunk order
    const long long base = (static_cast<long long>(t) * nh + hq) * a.max_chunks;
    float M = -INFINITY;
    for (int jj = 0; jj < nch; ++jj) M = fmaxf(M, __ldcg(a.part_ml + 2 * (base + jj)));
    float den = 0.f, acc[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] = 0.f;
    for (int jj = 0; jj < nch; ++jj) {
        const float wgt = __expf(__ldcg(a.part_ml + 2 * (base + jj)) - M);
        den = fmaf(__ldcg(a.part_ml + 2 * (base + jj) + 1), wgt, den);
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = fmaf(__ldcg(a.part_o + (base + jj) * HD + lane * DPL + e), wgt, acc[e]);
    }
    const float inv = 1.0f / den;
#pragma unroll
    for (int e = 0; e < DPL; ++e) out[e] = __float2bfloat16_rn(acc[e] * inv);
}

struct FwdSmem {
    uint64_t fullW[kFwdMaxStages], fullX[kFwdMaxStages], empty[kFwdMaxStages], tfull[2], tempty[2];
    unsigned long long ep;
    uint32_t tslot;
    int sint[12];
    float rs[256];
    float red[128];
    float sval[128];
    int sidx[128];
    float qv[512];
    float pv[256];
};
static_assert(sizeof(FwdSmem) <= kFwdMiscBytes, "misc shared state exceeds its budget");

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(kFwdThreads, 2) fwd_kernel(const __grid_constant__ FwdArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ FwdSmem sm;  // static: the compiler keeps these in the shared address space (LDS/STS)
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = a.stages, tp = a.tp;
    const int bbytes = tp * kBK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kABytes;
    uint64_t* fullW = sm.fullW;
    uint64_t* fullX = sm.fullX;
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
    float* qv = sm.qv;     // [4][128] attention query per warp
    float* pv = sm.pv;     // [4][64]  attention probabilities per warp

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x, G = gridDim.x;
    const uint32_t ncols = static_cast<uint32_t>(a.nacc * a.acc_cols);

    if (threadIdx.x == 0) {
        const LaneState* L = a.lane;
        const int start = min(L->kv_len, L->row0), Lc = L->L + L->c;
        sint[0] = start;
        sint[1] = Lc - start;
        sint[2] = Lc;
        *sep = *reinterpret_cast<volatile unsigned long long*>(a.epoch);
        for (int i = 0; i < S; ++i) {
            mbar_init(&fullW[i], 1);
            mbar_init(&fullX[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tslot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int start = sint[0], T = sint[1];
    const unsigned long long ep = *sep;
    if (T < 1 || T > tp) {  // host contract violated: nothing consistent to compute
        if (c == 0 && threadIdx.x == 0) {
            a.lane->error = 2;
            atomicExch(a.err, 100);
        }
        __syncthreads();
        if (warp == 1) tmem_dealloc(tmem, ncols);
        return;
    }

    if (warp == 0) {
        if (lane == 0) {  // ======================================================== TMA producer
            for (int i = 0; i < 5; ++i) tma_prefetch_desc(&a.wmaps[i]);
            for (int i = 0; i < 3; ++i) tma_prefetch_desc(&a.xmaps[i]);
            Cur w{}, x{};
            seek(w, a, c, G);
            seek(x, a, c, G);
            Ring wr, xr;
            if (a.simple_producer) {  // A/B reference: in-order, blocking (weights wait on dependencies)
                int dep_phase = -1;
                while (w.p < a.n_ph) {
                    mbar_wait_wd(&empty[wr.st], wr.ph ^ 1u, a.err, 1, w.p);
                    mbar_arrive_expect_tx(&fullW[wr.st], kABytes);
                    tma_load_2d(sA + wr.st * kABytes, &a.wmaps[w.wmap], &fullW[wr.st], w.kb * kBK, w.wrow + w.m * kBM,
                                kEvictFirst);
                    if (w.p != dep_phase) {
                        wait_dep(a, w.dep, ep, 1);
                        fence_proxy_async_global();
                        dep_phase = w.p;
                    }
                    mbar_arrive_expect_tx(&fullX[wr.st], bbytes);
                    for (int j = 0; j < tp / 16; ++j)
                        tma_load_2d(sB + wr.st * bbytes + j * 2048, &a.xmaps[w.xmap], &fullX[wr.st], w.kb * kBK, j * 16,
                                    kEvictLast);
                    wr.next(S);
                    step(w, a, c, G);
                }
            }
            int pending = 0;  // units whose weights are issued but whose activations are not
            int dep_phase = -1, stamped = -1;
            Spin spin;
            while (w.p < a.n_ph || pending > 0) {
                bool prog = false;
                if (pending > 0) {  // activations: only once the phase's input is complete
                    bool ok = x.p == dep_phase;
                    if (!ok && dep_ok(a, x.dep, ep)) {
                        fence_proxy_async_global();
                        dep_phase = x.p;
                        ok = true;
                        stamp(a, x.p, 1);
                    }
                    if (ok) {
                        if (a.dbg & 1) {
                            mbar_arrive(&fullX[xr.st]);
                        } else {
                            mbar_arrive_expect_tx(&fullX[xr.st], bbytes);
                            for (int j = 0; j < tp / 16; ++j)
                                tma_load_2d(sB + xr.st * bbytes + j * 2048, &a.xmaps[x.xmap], &fullX[xr.st],
                                            x.kb * kBK, j * 16, kEvictLast);
                        }
                        xr.next(S);
                        --pending;
                        step(x, a, c, G);
                        prog = true;
                    }
                }
                if (w.p < a.n_ph && mbar_test(&empty[wr.st], wr.ph ^ 1u)) {  // weights: as soon as a slot frees
                    if (stamped != w.p) {
                        stamp(a, w.p, 0);
                        stamped = w.p;
                    }
                    mbar_arrive_expect_tx(&fullW[wr.st], kABytes);
                    tma_load_2d(sA + wr.st * kABytes, &a.wmaps[w.wmap], &fullW[wr.st], w.kb * kBK, w.wrow + w.m * kBM,
                                kEvictFirst);
                    wr.next(S);
                    ++pending;
                    step(w, a, c, G);
                    prog = true;
                }
                if (prog) {
                    spin = Spin{};
                } else {
                    // Nothing issuable: park on the next ring slot (the hardware wakes the thread when it
                    // frees).  While activations wait on a dependency, bound the park so the flag is
                    // polled again within ~0.25 us.
                    spin.tick(a.err, 1, pending > 0 ? x.p : w.p);
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
            Ring rr, tr;  // smem ring; TMEM accumulator ring (nacc buffers)
            int mma_stamped = -1;
            while (k.p < a.n_ph) {
                const int p = k.p;
                const int n = min(k.e - k.u, k.KB - k.kb);  // units of this tile in this CTA's range
                mbar_wait_wd(&tempty[tr.st], tr.ph ^ 1u, a.err, 2, p);
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(tr.st * a.acc_cols);
                for (int i = 0; i < n; ++i) {
                    mbar_wait_wd(&fullW[rr.st], rr.ph, a.err, 3, p);
                    mbar_wait_wd(&fullX[rr.st], rr.ph, a.err, 4, p);
                    tc_fence_after();
                    if (p != mma_stamped) {
                        stamp(a, p, 4);  // first MMA of the phase
                        mma_stamped = p;
                    }
                    if (a.dbg & 2) {
                        mbar_arrive(&empty[rr.st]);
                    } else {
                        const uint64_t ad = umma_desc_sw128(smem_u32(sA + rr.st * kABytes));
                        const uint64_t bd = umma_desc_sw128(smem_u32(sB + rr.st * bbytes));
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk)
                            mma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc, (i > 0 || kk > 0) ? 1u : 0u);
                        mma_commit(&empty[rr.st]);
                    }
                    rr.next(S);
                    step(k, a, c, G);
                }
                if (a.dbg & 2) mbar_arrive(&tfull[tr.st]);
                else mma_commit(&tfull[tr.st]);
                tr.next(a.nacc);
                stamp(a, p, 5);  // last MMA issued (so far) for the phase
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
        {  // warm L2: this forward's embedding rows and RoPE rows (tiny, cold, on the critical path)
            const int gt = c * 128 + et, GT = G * 128;
            for (int t = gt; t < T; t += GT) l2_warm(a.embed + static_cast<long long>(a.buf[start + t]) * h, h * 2, 0, 1);
            if (gt == GT - 1) l2_warm(a.rope + static_cast<long long>(start) * (a.hd / 2), T * (a.hd / 2) * 8LL, 0, 1);
        }
        for (int p = 0; p < a.n_ph; ++p) {
            const FwdPhase& P = a.ph[p];
            if (P.kind == kPhGemm && P.epi == kFeQkv) {
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
                    const int tok = t < T ? a.buf[start + t] : 0;
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
                for (int u = rg.b0; u < rg.b1;) {
                    const int m = u / P.kb;
                    const int tile_u0 = m * P.kb, tile_u1 = tile_u0 + P.kb;
                    const int stop = min(tile_u1, rg.b1);
                    const int first = owner_of(tile_u0, U, A), last = owner_of(tile_u1 - 1, U, A);
                    const int n_contrib = static_cast<int>(last - first + 1);
                    const int my = static_cast<int>(rg.ci - first);
                    const int buf = it % a.nacc;
                    mbar_wait_wd(&tfull[buf], static_cast<uint32_t>((it / a.nacc) & 1), a.err, 6, p);
                    tc_fence_after();
                    if (et == 0) stamp(a, p, 7);  // accumulator of this CTA's latest tile ready
                    const uint32_t taddr = tmem + static_cast<uint32_t>(buf * a.acc_cols) + (static_cast<uint32_t>(q * 32) << 16);
                    bool finisher = true;
                    if (n_contrib > 1) {
                        const int slot = 2 * rg.ci + (u == rg.b0 ? 0 : 1);
                        float* Pp = a.ws + static_cast<long long>(slot) * tp * kBM;
                        for (int ch = 0; ch < tp; ch += 32) {
                            float v[32];
                            tmem_ld32(taddr + ch, v);
                            const int nc = min(32, tp - ch);
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (i < nc) __stcg(Pp + (ch + i) * kBM + r, v[i]);
                        }
                        named_bar_sync(1, 128);
                        if (et == 0) {  // one acq_rel RMW: releases our partial, acquires the others'
                            const bool last_in = atom_add_acq_rel_gpu(&a.tile_cnt[m], 1) == n_contrib - 1;
                            if (last_in) a.tile_cnt[m] = 0;  // reusable by the next split tile here
                            sint[3] = last_in;
                        }
                        named_bar_sync(1, 128);
                        finisher = sint[3] != 0;
                    }
                    if (et == 0 && finisher) stamp(a, p, 8);
                    if (finisher) {
                        const int n = m * kBM + r;
                        for (int ch = 0; ch < tp; ch += 32) {
                            float v[32];
                            tmem_ld32(taddr + ch, v);
                            const int nc = min(32, tp - ch);
                            if (n_contrib > 1) {  // ordered sum p_first + p_first+1 + ... (fixed per shape)
#pragma unroll
                                for (int g = 0; g < 32; g += 16) {
                                    if (g >= nc) break;
                                    float acc[16];
                                    for (int jb = 0; jb < n_contrib; jb += kBatch) {
                                        float x[kBatch][16];
#pragma unroll
                                        for (int j = 0; j < kBatch; ++j) {
                                            const int cj = first + jb + j;
                                            const int bj = range_begin(cj, U, A);
                                            const int slot = 2 * cj + (bj >= tile_u0 ? 0 : 1);
                                            const float* Pj = a.ws + static_cast<long long>(slot) * tp * kBM + (ch + g) * kBM + r;
                                            const bool load = jb + j < n_contrib && jb + j != my;
#pragma unroll
                                            for (int i = 0; i < 16; ++i)
                                                x[j][i] = (load && g + i < nc) ? __ldcg(Pj + i * kBM) : v[g + i];
                                        }
#pragma unroll
                                        for (int i = 0; i < 16; ++i) {
                                            float s2 = jb == 0 ? x[0][i] : acc[i] + x[0][i];
#pragma unroll
                                            for (int j = 1; j < kBatch; ++j)
                                                if (jb + j < n_contrib) s2 += x[j][i];
                                            acc[i] = s2;
                                        }
                                    }
#pragma unroll
                                    for (int i = 0; i < 16; ++i) v[g + i] = acc[i];
                                }
                            }
                            if (et == 0) stamp(a, p, 9);
                            // ---------------------------------------------- fused epilogues
                            if (P.epi == kFeResid) {
                                float sq[32];
                                float* o = a.resid + static_cast<long long>(ch) * h + n;
#pragma unroll
                                for (int i = 0; i < 32; ++i) sq[i] = i < nc ? __ldcg(o + static_cast<long long>(i) * h) : 0.f;
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    if (i < nc) {
                                        const float nv = sq[i] + v[i];
                                        o[static_cast<long long>(i) * h] = nv;
                                        a.xb[static_cast<long long>(ch + i) * h + n] = __float2bfloat16_rn(nv);
                                        sq[i] = nv * nv;
                                    }
                                }
                                red[q * 32 + lane] = warp_colsum32(sq, lane);
                                named_bar_sync(1, 128);
                                if (et < 32 && ch + et < tp)
                                    a.ssq[m * 256 + ch + et] = ((red[et] + red[32 + et]) + red[64 + et]) + red[96 + et];
                                named_bar_sync(1, 128);
                            } else if (P.epi == kFeSilu) {
                                const int f = m * 64 + q * 16 + lane;
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    const float x = i < nc ? v[i] * rs[ch + i] : 0.f;
                                    const float up = __shfl_down_sync(0xffffffffu, x, 16);
                                    if (lane < 16 && i < nc)
                                        a.act[static_cast<long long>(ch + i) * a.ffn_l + f] =
                                            __float2bfloat16_rn(x / (1.0f + __expf(-x)) * up);
                                }
                            } else if (P.epi == kFeQkv) {
                                const int hd = a.hd, half = hd >> 1;
                                const bool in_rows = n < P.n_out;  // warp-uniform (n_out % 64 == 0)
                                const bool is_q = n < a.q_dim, is_k = !is_q && n < a.q_dim + a.kv_dim;
                                const int base = is_q ? 0 : is_k ? a.q_dim : a.q_dim + a.kv_dim;
                                const int head = (n - base) / hd, pr = (n - base) % hd, qh = pr >> 5;
                                const int dd = lane < 16 ? 16 * qh + lane : half + 16 * qh + lane - 16;
                                const __nv_bfloat16* nw = is_q ? P.qn : is_k ? P.kn : nullptr;
                                const bool norm = in_rows && nw != nullptr && !(a.dbg & 4);
                                float x[32];
#pragma unroll
                                for (int i = 0; i < 32; ++i) x[i] = bf16r(v[i] * rs[ch + i]);
                                {
                                    float sq[32];
#pragma unroll
                                    for (int i = 0; i < 32; ++i) sq[i] = x[i] * x[i];
                                    red[q * 32 + lane] = warp_colsum32(sq, lane);
                                }
                                if (et == 0) stamp(a, p, 12);
                                named_bar_sync(1, 128);
                                if (et == 0) stamp(a, p, 13);
                                if (norm) {
                                    const int fq = q - qh, nwq = hd >> 5;
                                    const float wd = (a.dbg & 32) ? 1.0f : __bfloat162float(nw[dd]);
                                    const float inv_hd = 1.0f / static_cast<float>(hd);
#pragma unroll
                                    for (int i = 0; i < 32; ++i) {
                                        if (a.dbg & 64) break;
                                        float ss = red[fq * 32 + i];
                                        for (int w2 = 1; w2 < nwq; ++w2) ss += red[(fq + w2) * 32 + i];
                                        x[i] = bf16r(x[i] * rsqrtf(ss * inv_hd + a.eps) * wd);
                                    }
                                }
                                if (et == 0) stamp(a, p, 14);
                                named_bar_sync(1, 128);
                                if (et == 0) stamp(a, p, 15);
                                if (in_rows) {
                                    const int dm = dd % half;
                                    // RoPE partners, then every table load in flight before any store
#pragma unroll
                                    for (int i = 0; i < 32; ++i) {
                                        const float partner = __shfl_xor_sync(0xffffffffu, x[i], 16);
                                        if ((is_q || is_k) && !(a.dbg & 8)) {
                                            const float2 cs = ch + i < T ? __ldg(a.rope + static_cast<long long>(start + ch + i) * half + dm)
                                                                         : make_float2(1.f, 0.f);
                                            x[i] = lane < 16 ? x[i] * cs.x - partner * cs.y : x[i] * cs.x + partner * cs.y;
                                        }
                                    }
                                    if (a.dbg & 16) {
                                    } else if (is_q) {
                                        __nv_bfloat16* dq = a.qbuf + (static_cast<long long>(ch) * a.nh + head) * hd + dd;
#pragma unroll
                                        for (int i = 0; i < 32; ++i)
                                            if (ch + i < T) dq[static_cast<long long>(i) * a.nh * hd] = __float2bfloat16_rn(x[i]);
                                    } else {
                                        __nv_bfloat16* kvc = is_k ? P.kc : P.vc;
                                        int pg[32];
#pragma unroll
                                        for (int i = 0; i < 32; ++i)
                                            pg[i] = ch + i < T ? __ldg(a.page_table + (start + ch + i) / kPage) : 0;
#pragma unroll
                                        for (int i = 0; i < 32; ++i) {
                                            const int pos = start + ch + i;
                                            if (ch + i < T)
                                                kvc[((static_cast<long long>(pg[i]) * a.nkv + head) * kPage + pos % kPage) * hd + dd] =
                                                    __float2bfloat16_rn(x[i]);
                                        }
                                    }
                                }
                            } else {  // kFeLogits: scaled logits, per-tile (max, lowest index) per column
                                const bool ok = n < P.n_out;
#pragma unroll
                                for (int i = 0; i < 32; ++i) v[i] *= rs[ch + i];
                                if (a.logits && ok) {
#pragma unroll
                                    for (int i = 0; i < 32; ++i)
                                        if (i < nc && ch + i < T) a.logits[static_cast<long long>(ch + i) * a.ld_logits + n] = v[i];
                                }
#pragma unroll
                                for (int i = 0; i < 32; ++i) {
                                    float bv = ok ? v[i] : -INFINITY;
                                    int bi = ok ? n : 0x7fffffff;
#pragma unroll
                                    for (int off = 16; off > 0; off >>= 1) {
                                        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                                        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                                        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                                    }
                                    if (lane == i) { sval[q * 32 + i] = bv; sidx[q * 32 + i] = bi; }
                                }
                                named_bar_sync(1, 128);
                                if (et < 32 && et < nc) {
                                    float bv = sval[et];
                                    int bi = sidx[et];
                                    for (int qq = 1; qq < 4; ++qq) {
                                        const float ov = sval[qq * 32 + et];
                                        const int oi = sidx[qq * 32 + et];
                                        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                                    }
                                    a.amax[static_cast<long long>(m) * tp + ch + et] = make_float2(bv, __int_as_float(bi));
                                }
                                named_bar_sync(1, 128);
                            }
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
                const int nh = a.nh;
                const int nch_max = (start + T - 1) / kAttnChunk + 1;
                const int items = T * nh * nch_max;
                float* q_s = qv + ew * 128;
                float* p_s = pv + ew * 64;
                for (int item = gw; item < items; item += GW) {
                    const int j = item % nch_max, rest = item / nch_max;
                    const int hq = rest % nh, t = rest / nh;
                    if (j * kAttnChunk > start + t) continue;
                    if (a.hd == 128) attn_item<128>(a, P, t, hq, j, start, q_s, p_s, lane);
                    else attn_item<64>(a, P, t, hq, j, start, q_s, p_s, lane);
                }
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
                    if (lane == 0) a.argmax[start + t] = (bi == 0x7fffffff || bv != bv) ? -1 : bi;
                }
                signal(p);
                if (c == 0 && et == 0) {  // the forward is complete once every CTA has signalled
                    wait_dep(a, p, ep, 7);
                    a.lane->start = start;
                    a.lane->kv_len = sint[2];
                    __threadfence();
                    *reinterpret_cast<volatile unsigned long long*>(a.epoch) = ep + 1;
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

bool fwd_simple_producer() {
    static const bool on = [] {
        const char* e = std::getenv("DBL_FWD_SIMPLE");
        return e && e[0] == '1';
    }();
    return on;
}

void fwd_prepare() {
    static std::once_flag once;
    std::call_once(once, [] {
        CUDA_CHECK(cudaFuncSetAttribute(fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - kFwdMiscBytes));
    });
}

int fwd_smem_budget() {  // DBL_FWD_SMEM_KB overrides (A/B)
    static const int kb = [] {
        const char* e = std::getenv("DBL_FWD_SMEM_KB");
        return e ? std::atoi(e) : 0;
    }();
    return kb > 0 ? std::min(kb, 227) * 1024 : kFwdSmemBudget;
}

int fwd_stages(int tp, size_t* smem) {
    const int stage = kABytes + tp * kBK * 2;
    const int s = (fwd_smem_budget() - 1024 - kFwdMiscBytes) / stage;  // kFwdMiscBytes: the static FwdSmem
    if (s < 2) throw_invalid("stream forward: token bucket too large for the shared-memory ring");
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

void fwd_launch(const FwdArgs& a, int grid, size_t smem, cudaStream_t s) {
    fwd_prepare();
    fwd_kernel<<<grid, kFwdThreads, smem, s>>>(a);
    CUDA_LAUNCH_CHECK();
}

}  // namespace dbl
