// Weight-stream ceiling probe: how fast can persistent CTAs pull contiguous stream-K unit ranges of
// 16 KiB weight tiles into a shared-memory ring (no math)?  Compares the forward's 2D TMA box
// (128 rows x 64 k of a row-major [N][K] matrix) with a 1D bulk copy of a pre-tiled, contiguous
// 16 KiB image.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/stream_probe tools/stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2601_05524_b200/csrc/sm100.cuh"

using namespace dbl::sm100;

constexpr int kTile = 128 * 64 * 2;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t hint) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(hint)
        : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                    const __grid_constant__ CUtensorMap xmap, const uint8_t* w, int U,
                                                    int KB, int S, int tiles_per_copy, int busy) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[32], empty[32];
    const int ci = blockIdx.x, A = gridDim.x;
    const int b0 = static_cast<int>(static_cast<long long>(ci) * U / A);
    const int b1 = static_cast<int>(static_cast<long long>(ci + 1) * U / A);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int step = MODE == 1 ? tiles_per_copy : 1;
    const int xb = MODE == 3 ? 16 * 64 * 2 : 0;  // MODE 3: tiled weights + a 16-row activation box per stage
    if (threadIdx.x == 0) {  // producer
        int st = 0, ph = 0;
        for (int u = b0; u < b1; u += step) {
            mbar_wait(&empty[st], ph ^ 1);
            if (busy) {  // emulate per-stage producer bookkeeping
                const long long t0 = clock64();
                while (clock64() - t0 < busy) {}
            }
            const int n = min(step, b1 - u);
            mbar_arrive_expect_tx(&full[st], n * kTile + xb);
            uint8_t* dst = smem + static_cast<size_t>(st) * step * (kTile + xb);
            if (MODE == 3) tma_load_2d(dst + kTile, &xmap, &full[st], (u % KB) * 64, 0, kEvictLast);
            if (MODE == 0) tma_load_2d(dst, &map, &full[st], (u % KB) * 64, (u / KB) * 128, kEvictFirst);
            else if (MODE >= 2) tma_load_2d(dst, &map, &full[st], 0, u * 128, kEvictFirst);  // tiled [U*128][64] view
            else bulk_g2s(dst, w + static_cast<size_t>(u) * kTile, n * kTile, &full[st], kEvictFirst);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {  // consumer
        int st = 0, ph = 0;
        for (int u = b0; u < b1; u += step) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long K = 5120, N = 104832;  // ~1 GiB of bf16
    const size_t bytes = static_cast<size_t>(N) * K * 2;
    uint8_t* w;
    cudaMalloc(&w, bytes);
    cudaMemset(w, 1, bytes);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap map, tmap;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K * 2)};
    const cuuint32_t box[2] = {64, 128}, estr[2] = {1, 1};
    reinterpret_cast<EncodeFn>(p)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    {
        const cuuint64_t d2[2] = {64, static_cast<cuuint64_t>(N * K / 64)};
        const cuuint64_t s2[1] = {128};
        reinterpret_cast<EncodeFn>(p)(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, d2, s2, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    CUtensorMap xm;
    uint8_t* x;
    cudaMalloc(&x, 16 * K * 2);
    cudaMemset(x, 0, 16 * K * 2);
    {
        const cuuint64_t d2[2] = {static_cast<cuuint64_t>(K), 16};
        const cuuint64_t s2[1] = {static_cast<cuuint64_t>(K * 2)};
        const cuuint32_t b2[2] = {64, 16};
        reinterpret_cast<EncodeFn>(p)(&xm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, d2, s2, b2, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const int KB = static_cast<int>(K / 64), U = static_cast<int>(N / 128) * KB;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int mode, per_sm, S, tpc, busy; };
    const Cfg cfgs[] = {{3, 1, 5, 1, 0},   {3, 1, 5, 1, 200},  {3, 1, 5, 1, 400}, {3, 1, 5, 1, 600},
                        {3, 1, 5, 1, 800}, {3, 1, 5, 1, 1000}, {3, 2, 5, 1, 400}, {3, 2, 5, 1, 800}};
    for (const Cfg& c : cfgs) {
        const int grid = sms * c.per_sm;
        const size_t sm_bytes = static_cast<size_t>(c.S) * c.tpc * (kTile + (c.mode == 3 ? 2048 : 0));
        float best = 1e30f, sum = 0.f;
        const int reps = 20;
        for (int r = 0; r < reps + 2; ++r) {
            cudaEventRecord(e0);
            if (c.mode == 0) stream_kernel<0><<<grid, 64, sm_bytes>>>(map, xm, w, U, KB, c.S, c.tpc, c.busy);
            else if (c.mode == 1) stream_kernel<1><<<grid, 64, sm_bytes>>>(map, xm, w, U, KB, c.S, c.tpc, c.busy);
            else if (c.mode == 2) stream_kernel<2><<<grid, 64, sm_bytes>>>(tmap, xm, w, U, KB, c.S, c.tpc, c.busy);
            else stream_kernel<3><<<grid, 64, sm_bytes>>>(tmap, xm, w, U, KB, c.S, c.tpc, c.busy);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
        }
        const cudaError_t err = cudaGetLastError();
        printf("busy=%d mode=%s ctas/sm=%d stages=%d tiles/copy=%d smem=%zuKB: best %.1f GB/s mean %.1f GB/s %s\n",
               c.busy, c.mode == 0 ? "tma2d" : c.mode == 1 ? "bulk1d" : c.mode == 2 ? "tma2d-tiled" : "tiled+x", c.per_sm, c.S, c.tpc, sm_bytes / 1024, bytes / best / 1e6,
               bytes / (sum / reps) / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    return 0;
}
