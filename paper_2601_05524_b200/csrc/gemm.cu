// tcgen05 swap-AB stream-K GEMM (see gemm.cuh for the design).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "gemm.cuh"
#include "lane.cuh"
#include "launch.cuh"
#include "sm100.cuh"

namespace dbl {

namespace {

constexpr int kThreads = 192;  // warp0 TMA, warp1 MMA, warps 2..5 epilogue
constexpr int kBlockM = 128, kBlockK = 64;
constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KiB
constexpr int kMaxBatchContrib = 8;             // split-K fan-in reduced with batched loads

__device__ __forceinline__ long long range_begin(long long c, long long U, long long G) { return c * U / G; }
// CTA whose range contains unit u: largest c with floor(cU/G) <= u
__device__ __forceinline__ long long cta_of(long long u, long long U, long long G) {
    return ((u + 1) * G - 1) / U;
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmN, GemmArgs a) {
    using namespace sm100;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = a.stages, tp = a.tp;
    const int b_bytes = tp * kBlockK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * b_bytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
    int* sflag = reinterpret_cast<int*>(tslot + 1);
    float* sval = reinterpret_cast<float*>(sflag + 4);  // [4][32]
    int* sidx = reinterpret_cast<int*>(sval + 128);     // [4][32]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long U = a.units, G = gridDim.x, c = blockIdx.x;
    const long long b0 = range_begin(c, U, G), b1 = range_begin(c + 1, U, G);
    if (b0 >= b1) return;
    const int KB = a.kb_total;
    const uint32_t ncols = tp <= 32 ? 32 : tp <= 64 ? 64 : tp <= 128 ? 128 : 256;
    auto stamp = [&](int k) {
        if (a.trace) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[c * 4 + k] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);  // CTA resident

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 128);
        fence_barrier_init();
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
    }
    if (warp == 1) tmem_alloc(tslot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    griddep_launch_dependents();  // PDL: the next kernel may start its prologue / weight prefetch

    if (warp == 0) {
        if (lane == 0) {  // ------------------------------------------------ TMA producer
            // The weights never depend on the previous kernel: prefetch the first S stages' weight
            // tiles BEFORE the grid-dependency wait (overlapping the previous kernel's tail), then
            // wait and fetch the activation tiles.
            const long long n_units = b1 - b0;
            const int pre = static_cast<int>(std::min<long long>(S, n_units));
            for (int i = 0; i < pre; ++i) {
                const long long u = b0 + i;
                mbar_arrive_expect_tx(&full[i], kABytes + b_bytes);
                tma_load_2d(sA + i * kABytes, &tmW, &full[i], static_cast<int>(u % KB) * kBlockK,
                            static_cast<int>(u / KB) * kBlockM, kEvictFirst);
            }
            // ...and warm L2 with the rest of this CTA's weight range (bounded so one GEMM's warm set
            // stays well inside the 126 MB L2): HBM keeps streaming while the previous kernels of the
            // forward drain, instead of idling at the kernel boundary.
            const long long pf_end = std::min<long long>(b1, b0 + pre + a.l2_prefetch_units);
            for (long long u = b0 + pre; u < pf_end; ++u)
                tma_prefetch_l2_2d(&tmW, static_cast<int>(u % KB) * kBlockK, static_cast<int>(u / KB) * kBlockM);
            griddep_wait();
            stamp(1);  // dependency resolved
            for (int i = 0; i < pre; ++i) {
                const int kb = static_cast<int>((b0 + i) % KB);
                for (int j = 0; j < tp / 16; ++j)
                    tma_load_2d(sB + i * b_bytes + j * 2048, &tmX, &full[i], kb * kBlockK, j * 16, kEvictLast);
            }
            int stage = pre % S;
            uint32_t phase = pre == S ? 1u : 0u;
            for (long long u = b0 + pre; u < b1; ++u) {
                const int m = static_cast<int>(u / KB), kb = static_cast<int>(u % KB);
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_arrive_expect_tx(&full[stage], kABytes + b_bytes);
                tma_load_2d(sA + stage * kABytes, &tmW, &full[stage], kb * kBlockK, m * kBlockM, kEvictFirst);
                for (int j = 0; j < tp / 16; ++j)
                    tma_load_2d(sB + stage * b_bytes + j * 2048, &tmX, &full[stage], kb * kBlockK, j * 16,
                                kEvictLast);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            stamp(2);  // last load issued
            // Warm L2 with the NEXT GEMM's first weight tiles (those of the CTA at the same relative
            // grid position): HBM keeps streaming through this GEMM's drain and through the small
            // dependent kernels (norm / RoPE / attention) that separate it from the next one.
            if (a.next_units > 0) {
                const long long G2 = a.next_grid, U2 = a.next_units, c2 = c * G2 / G;
                const long long s2 = range_begin(c2, U2, G2);
                const long long e2 = std::min<long long>(range_begin(c2 + 1, U2, G2), s2 + a.next_prefetch);
                for (long long u = s2; u < e2; ++u)
                    tma_prefetch_l2_2d(&tmN, static_cast<int>(u % a.next_kb) * kBlockK,
                                       static_cast<int>(u / a.next_kb) * kBlockM);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ------------------------------------------------ MMA issuer
            const uint32_t idesc = idesc_bf16_m128(tp);
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (long long u = b0; u < b1;) {
                const int kb0 = static_cast<int>(u % KB);
                const int kb1 = static_cast<int>(std::min<long long>(KB, kb0 + (b1 - u)));
                mbar_wait(tempty, acc_phase ^ 1);
                tc_fence_after();
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = umma_desc_sw128(smem_u32(sA + stage * kABytes));
                    const uint64_t bd = umma_desc_sw128(smem_u32(sB + stage * b_bytes));
#pragma unroll
                    for (int k = 0; k < kBlockK / 16; ++k)
                        mma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    mma_commit(&empty[stage]);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                mma_commit(tfull);
                acc_phase ^= 1;
                u += kb1 - kb0;
            }
        }
    } else {  // ------------------------------------------------------------ epilogue (128 threads)
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int r = q * 32 + lane;
        const int et = threadIdx.x - 64;  // 0..127
        const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
        uint32_t acc_phase = 0;
        for (long long u = b0; u < b1;) {
            const int m = static_cast<int>(u / KB), kb0 = static_cast<int>(u % KB);
            const int kb1 = static_cast<int>(std::min<long long>(KB, kb0 + (b1 - u)));
            const long long tile_u0 = static_cast<long long>(m) * KB, tile_u1 = tile_u0 + KB;
            const long long first = cta_of(tile_u0, U, G), last = cta_of(tile_u1 - 1, U, G);
            const int n_contrib = static_cast<int>(last - first + 1);
            const int my = static_cast<int>(c - first);
            mbar_wait(tfull, acc_phase);
            tc_fence_after();
            bool finisher = true;
            if (n_contrib > 1) {
                const int slot = static_cast<int>(2 * c + (u == b0 ? 0 : 1));
                float* P = a.ws + static_cast<long long>(slot) * tp * kBlockM;
                for (int ch = 0; ch < tp; ch += 32) {
                    float v[32];
                    tmem_ld32(taddr + ch, v);
                    const int nc = min(32, tp - ch);
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < nc) __stcg(P + (ch + i) * kBlockM + r, v[i]);
                }
                // publish: CTA barrier, then ONE gpu-scope fence + arrival (semaphore pattern)
                named_bar_sync(1, 128);
                if (et == 0) {
                    __threadfence();
                    const bool last_in = atomicAdd(&a.counters[m], 1) == n_contrib - 1;
                    if (last_in) {
                        __threadfence();     // acquire the other contributors' partials
                        a.counters[m] = 0;   // reusable by the next launch
                    }
                    sflag[0] = last_in;
                }
                named_bar_sync(1, 128);
                finisher = sflag[0] != 0;
            }
            if (finisher) {
                for (int ch = 0; ch < tp; ch += 32) {
                    float v[32];
                    tmem_ld32(taddr + ch, v);
                    const int nc = min(32, tp - ch);
                    if (n_contrib > 1 && n_contrib <= kMaxBatchContrib) {
                        // ordered sum p_0 + p_1 + ... with every contributor's loads of an 8-column
                        // group in flight at once (one L2 round trip per group)
                        const float* Pj[kMaxBatchContrib];
#pragma unroll
                        for (int j = 0; j < kMaxBatchContrib; ++j) {
                            const long long cj = first + j;
                            const long long bj = range_begin(cj, U, G);
                            const int slot = static_cast<int>(2 * cj + (std::max(bj, tile_u0) == bj ? 0 : 1));
                            Pj[j] = a.ws + static_cast<long long>(slot) * tp * kBlockM + ch * kBlockM + r;
                        }
#pragma unroll
                        for (int g8 = 0; g8 < 32; g8 += 8) {
                            if (g8 >= nc) break;
                            float x[kMaxBatchContrib][8];
#pragma unroll
                            for (int j = 0; j < kMaxBatchContrib; ++j)
#pragma unroll
                                for (int i = 0; i < 8; ++i)
                                    x[j][i] = (j < n_contrib && j != my && g8 + i < nc)
                                                  ? __ldcg(Pj[j] + (g8 + i) * kBlockM) : v[g8 + i];
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                float s = x[0][i];
#pragma unroll
                                for (int j = 1; j < kMaxBatchContrib; ++j)
                                    if (j < n_contrib) s += x[j][i];
                                v[g8 + i] = s;
                            }
                        }
                    } else if (n_contrib > 1) {  // ordered sum p_0 + p_1 + ... (fixed for every token count)
                        float acc[32];
                        for (int j = 0; j < n_contrib; ++j) {
                            const long long cj = first + j;
                            const long long bj = range_begin(cj, U, G);
                            const int slot = static_cast<int>(2 * cj + (std::max(bj, tile_u0) == bj ? 0 : 1));
                            const float* P = a.ws + static_cast<long long>(slot) * tp * kBlockM + ch * kBlockM + r;
                            float x[32];
                            if (j == my) {
#pragma unroll
                                for (int i = 0; i < 32; ++i) x[i] = v[i];
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; ++i) x[i] = i < nc ? __ldcg(P + i * kBlockM) : 0.f;
                            }
#pragma unroll
                            for (int i = 0; i < 32; ++i) acc[i] = j == 0 ? x[i] : acc[i] + x[i];
                        }
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = acc[i];
                    }
                    const int n = m * kBlockM + r;
                    if constexpr (EPI == static_cast<int>(Epi::StoreBF16)) {
                        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + static_cast<long long>(ch) * a.ld_out + n;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nc) o[static_cast<long long>(i) * a.ld_out] = __float2bfloat16_rn(v[i]);
                    } else if constexpr (EPI == static_cast<int>(Epi::StoreF32)) {
                        float* o = static_cast<float*>(a.out) + static_cast<long long>(ch) * a.ld_out + n;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nc) o[static_cast<long long>(i) * a.ld_out] = v[i];
                    } else if constexpr (EPI == static_cast<int>(Epi::ResidAdd)) {
                        float* o = static_cast<float*>(a.out) + static_cast<long long>(ch) * a.ld_out + n;
                        float old[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) old[i] = i < nc ? o[static_cast<long long>(i) * a.ld_out] : 0.f;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nc) o[static_cast<long long>(i) * a.ld_out] = old[i] + v[i];
                    } else if constexpr (EPI == static_cast<int>(Epi::SiluMul)) {
                        __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out);
                        const int f = m * 64 + q * 16 + lane;
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const float up = __shfl_down_sync(0xffffffffu, v[i], 16);
                            if (lane < 16 && i < nc) {
                                const float g = v[i];
                                o[static_cast<long long>(ch + i) * a.ld_out + f] =
                                    __float2bfloat16_rn(g / (1.0f + __expf(-g)) * up);
                            }
                        }
                    } else {  // Argmax
                        const bool ok = n < a.n_valid;
                        if (a.logits && ok) {  // only the forward's valid rows (the buffer holds no padding)
                            const int nrow = a.lane ? a.lane->L + a.lane->c - a.lane->start : tp;
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (i < nc && ch + i < nrow) a.logits[static_cast<long long>(ch + i) * a.ld_logits + n] = v[i];
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
                            a.amax_ws[static_cast<long long>(m) * tp + ch + et] = make_float2(bv, __int_as_float(bi));
                        }
                        named_bar_sync(1, 128);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty);
            acc_phase ^= 1;
            u += kb1 - kb0;
        }
        if (et == 0) stamp(3);  // epilogue done
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, ncols);
    }
}

// one warp per token row: reduce the per-tile (max, lowest idx) partials in tile order
__global__ void argmax_finish_kernel(const float2* __restrict__ ws, int n_tiles, int tp, const LaneState* lane,
                                     int32_t* __restrict__ argmax) {
    sm100::griddep_launch_dependents();
    sm100::griddep_wait();
    const int start = lane->start;
    const int T = lane->L + lane->c - start;
    const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int ln = threadIdx.x & 31;
    if (t >= T || t >= tp) return;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int m = ln; m < n_tiles; m += 32) {
        const float2 p = ws[static_cast<long long>(m) * tp + t];
        const int pi = __float_as_int(p.y);
        if (p.x > bv || (p.x == bv && pi < bi)) { bv = p.x; bi = pi; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (ln == 0) argmax[start + t] = (bi == 0x7fffffff || bv != bv) ? -1 : bi;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(DBL_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

template <int EPI>
void set_smem_attr() {
    static std::once_flag once;
    std::call_once(once, [] {
        CUDA_CHECK(cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    });
}

}  // namespace

int num_sms(int device) {
    static int cache[64] = {0};
    if (device >= 0 && device < 64 && cache[device]) return cache[device];
    int n = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    if (device >= 0 && device < 64) cache[device] = n;
    return n;
}

GemmTrace& gemm_trace() {
    static GemmTrace t;
    return t;
}

void gemm_prepare() {
    set_smem_attr<static_cast<int>(Epi::StoreBF16)>();
    set_smem_attr<static_cast<int>(Epi::ResidAdd)>();
    set_smem_attr<static_cast<int>(Epi::SiluMul)>();
    set_smem_attr<static_cast<int>(Epi::Argmax)>();
    set_smem_attr<static_cast<int>(Epi::StoreF32)>();
}

CUtensorMap make_tmap_bf16_tiled(const void* ptr, uint64_t tiles) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kBlockK), tiles * 128};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kBlockK) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockK), 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(DBL_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

CUtensorMap make_tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockK), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    if (cols % kBlockK) throw_invalid("GEMM K must be a multiple of 64");
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(DBL_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

CUtensorMap make_tmap_bf16_kblocks(const void* ptr, uint64_t rows, uint64_t cols, int box_rows, int box_kb) {
    // [rows][cols] K-major viewed as (64 elements, row, k-block): one box = box_kb consecutive 64-wide
    // k-blocks of box_rows rows, laid out in shared memory as box_kb stacked [box_rows][64] SW128 tiles
    CUtensorMap m;
    if (cols % kBlockK) throw_invalid("GEMM K must be a multiple of 64");
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kBlockK), rows, cols / kBlockK};
    const cuuint64_t strides[2] = {cols * 2, static_cast<cuuint64_t>(kBlockK) * 2};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(kBlockK), static_cast<cuuint32_t>(box_rows),
                               static_cast<cuuint32_t>(box_kb)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(DBL_CUDA_ERROR, "cuTensorMapEncodeTiled (k-block view) failed: " + std::to_string(r));
    return m;
}

void GemmWorkspace::ensure(int sms, int mtp, int mtiles) {
    const int g = 2 * sms + kMaxBatchContrib;  // split-K grids reach tiles * S < sms + tiles * 1
    if (g <= grid && mtp <= max_tp && mtiles <= max_tiles) return;
    grid = std::max(grid, g);
    max_tp = std::max(max_tp, mtp);
    max_tiles = std::max(max_tiles, mtiles);
    partials.alloc(static_cast<size_t>(2) * grid * max_tp * kBlockM);
    counters.alloc(max_tiles);
    counters.zero();
    amax.alloc(static_cast<size_t>(max_tiles) * max_tp);
    CUDA_CHECK(cudaDeviceSynchronize());
}

namespace {
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
// Grid = a pure function of (n_tiles, k-blocks, #SMs) — never of the token count — so the split
// points (and the numerics) are identical for every forward size.  Few tiles: regular split-K with
// S aligned slices per tile (S = ceil(SMs / tiles) <= 8 = the fan-in the finisher reduces with
// batched loads; two CTAs fit per SM).  Many tiles: stream-K over one CTA per SM.
int choose_grid(int n_tiles, int kb_total, int sms) {
    long long grid;
    if (n_tiles >= sms) {
        grid = sms;
    } else {
        const int S = std::min({kMaxBatchContrib, (sms + n_tiles - 1) / n_tiles, kb_total});
        grid = static_cast<long long>(n_tiles) * S;
    }
    return static_cast<int>(std::min<long long>(grid, static_cast<long long>(n_tiles) * kb_total));
}
}  // namespace

void gemm_launch(Epi epi, const CUtensorMap& tmW, const CUtensorMap& tmX, int n_out, int K, int tp, int n_valid,
                 void* out, int ld_out, float* logits, int ld_logits, GemmWorkspace& ws, cudaStream_t s,
                 const LaneState* lane, const GemmNext* next) {
    if (tp < 16 || tp > 256 || tp % 16) throw_invalid("GEMM token tile must be a multiple of 16 in [16, 256]");
    if (K % kBlockK) throw_invalid("GEMM K must be a multiple of 64");
    GemmArgs a{};
    a.n_out = n_out;
    a.K = K;
    a.tp = tp;
    a.n_valid = n_valid;
    a.n_tiles = (n_out + kBlockM - 1) / kBlockM;
    a.kb_total = K / kBlockK;
    a.units = static_cast<long long>(a.n_tiles) * a.kb_total;
    const int stage_bytes = kABytes + tp * kBlockK * 2;
    // decode-sized forwards (tp <= 64): ~110 KB so two GEMM CTAs (consecutive kernels under PDL)
    // co-reside on an SM; prefill-sized forwards take the whole SM for a deeper pipeline.
    // DBL_GEMM_STAGES overrides (tuning).
    // Long stream-K GEMMs (>= 64 k-blocks per CTA: gate|up, LM head) are pure streaming and take the
    // whole SM for 12 stages; split-K GEMMs keep two CTAs per SM.
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    const int sms = num_sms(dev);
    const int grid = choose_grid(a.n_tiles, a.kb_total, sms);
    static const int stage_cap = env_int("DBL_GEMM_STAGES", 0);
    const bool deep = stage_cap > 0 || tp > 64 || a.units / grid >= 64;
    const int budget = (deep ? 227 * 1024 : 110 * 1024) - 1024 - 2048;
    a.stages = std::max(2, std::min(stage_cap > 0 ? stage_cap : 12, budget / stage_bytes));
    const size_t smem = 1024 + static_cast<size_t>(a.stages) * stage_bytes + 2048;
    // DBL_GEMM_L2PF_MB: L2 warm-up of this GEMM's own later k-blocks before the dependency wait
    // and DBL_GEMM_NEXT_MB: warm-up of the next GEMM's first k-blocks after this one has issued its
    // last load.  Both measured slower in the full forward (the HBM is already busy during those
    // windows; see profiles/): off by default, kept for A/B runs.
    static const long long own_pf = static_cast<long long>(env_int("DBL_GEMM_L2PF_MB", 0)) << 20;
    static const long long next_pf = static_cast<long long>(env_int("DBL_GEMM_NEXT_MB", 0)) << 20;
    a.l2_prefetch_units = static_cast<int>(own_pf / (static_cast<long long>(kABytes) * grid));
    CUtensorMap tmN = tmW;
    if (next && next_pf > 0) {
        const int nt = (next->n_out + kBlockM - 1) / kBlockM, nkb = next->K / kBlockK;
        a.next_units = static_cast<long long>(nt) * nkb;
        a.next_grid = choose_grid(nt, nkb, sms);
        a.next_kb = nkb;
        a.next_prefetch = static_cast<int>(next_pf / (static_cast<long long>(kABytes) * a.next_grid));
        tmN = *next->tmap;
    }
    static const bool tracing = env_int("DBL_GEMM_TRACE", 0) != 0;
    if (tracing) {
        GemmTrace& tr = gemm_trace();
        if (!tr.buf.p) tr.buf.alloc(static_cast<size_t>(kTraceLaunches) * kTraceCtas * 4);
        if (tr.n < kTraceLaunches && grid <= kTraceCtas) {
            a.trace = tr.buf.p + static_cast<size_t>(tr.n) * kTraceCtas * 4;
            tr.grid.push_back(grid);
            tr.bytes.push_back(static_cast<long long>(n_out) * K * 2);
            ++tr.n;
        }
    }
    if (ws.grid < grid || ws.max_tp < tp || ws.max_tiles < a.n_tiles)
        throw_runtime("GEMM workspace too small (call GemmWorkspace::ensure)");
    a.out = out;
    a.ld_out = ld_out;
    a.logits = logits;
    a.ld_logits = ld_logits;
    a.lane = lane;
    a.amax_ws = ws.amax.p;
    a.ws = ws.partials.p;
    a.counters = ws.counters.p;
    switch (epi) {
#define DBL_GEMM_CASE(E)                                                                     \
    case E:                                                                                  \
        set_smem_attr<static_cast<int>(E)>();                                                \
        launch_pdl(gemm_kernel<static_cast<int>(E)>, dim3(grid), dim3(kThreads), smem, s, tmW, tmX, tmN, a); \
        break;
        DBL_GEMM_CASE(Epi::StoreBF16)
        DBL_GEMM_CASE(Epi::ResidAdd)
        DBL_GEMM_CASE(Epi::SiluMul)
        DBL_GEMM_CASE(Epi::Argmax)
        DBL_GEMM_CASE(Epi::StoreF32)
#undef DBL_GEMM_CASE
    }
}

void argmax_finish(const GemmWorkspace& ws, int n_tiles, int tp, const LaneState* lane, int32_t* argmax,
                   cudaStream_t s) {
    launch_pdl(argmax_finish_kernel, dim3((tp + 7) / 8), dim3(256), 0, s, static_cast<const float2*>(ws.amax.p),
               n_tiles, tp, lane, argmax);
}

}  // namespace dbl
