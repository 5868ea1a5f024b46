// Transformer set-up kernels (see tf_kernels.cuh): seeded weight init and tiled weight images.
#include <algorithm>
#include <cmath>

#include "tf_kernels.cuh"

namespace dbl {

namespace {

__host__ __device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d49bb133111ebull;
    return x ^ (x >> 31);
}
// N(0,1) from a 64-bit counter hash (Box-Muller on two 24-bit uniforms)
__device__ __forceinline__ float normal_of(unsigned long long key) {
    const unsigned long long h = mix(key);
    const float u1 = (static_cast<float>(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = static_cast<float>((h >> 16) & 0xFFFFFFull) * (1.0f / 16777216.0f);
    return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

__global__ void init_normal_kernel(__nv_bfloat16* dst, int rows, int cols, int ld, unsigned long long base,
                                   long long r0, long long c0, long long C, float std) {
    const long long n = static_cast<long long>(rows) * cols;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = i / cols, cc = i % cols;
        const long long logical = (r0 + r) * C + (c0 + cc);
        dst[r * ld + cc] = __float2bfloat16_rn(std * normal_of(base ^ static_cast<unsigned long long>(logical)));
    }
}

__global__ void init_gateup_kernel(__nv_bfloat16* dst, int ffn_local, int hidden, unsigned long long gbase,
                                   unsigned long long ubase, long long f0, float std) {
    const long long n = 2LL * ffn_local * hidden;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / hidden, col = i % hidden;
        // physical row p: tile j = p/128, quadrant q = (p%128)/32, half = (p%32)/16, lane = p%16
        const long long j = p / 128, q = (p % 128) / 32, half = (p % 32) / 16, ln = p % 16;
        const long long f = f0 + j * 64 + q * 16 + ln;  // logical ffn feature
        const unsigned long long base = half ? ubase : gbase;
        dst[i] = __float2bfloat16_rn(std * normal_of(base ^ static_cast<unsigned long long>(f * hidden + col)));
    }
}

// fused [q; k; v] projection with the rows of every head permuted so that RoPE partners share a warp:
// physical head row 32*w + l holds logical dim 16*w + l (l < 16) or hd/2 + 16*w + (l - 16) (l >= 16)
__global__ void init_qkv_kernel(__nv_bfloat16* dst, int q_dim, int kv_dim, int hd, int hidden,
                                unsigned long long qb, unsigned long long kb, unsigned long long vb, long long rq0,
                                long long rkv0, float std) {
    const long long rows = q_dim + 2LL * kv_dim;
    const long long n = rows * hidden;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / hidden, col = i % hidden;
        const int region = p < q_dim ? 0 : p < q_dim + kv_dim ? 1 : 2;
        const long long pl = p - (region == 0 ? 0 : region == 1 ? q_dim : q_dim + kv_dim);
        const long long head = pl / hd, pr = pl % hd, w = pr / 32, l = pr % 32;
        const long long dd = l < 16 ? 16 * w + l : hd / 2 + 16 * w + l - 16;
        const long long logical_row = (region == 0 ? rq0 : rkv0) + head * hd + dd;
        const unsigned long long base = region == 0 ? qb : region == 1 ? kb : vb;
        dst[i] = __float2bfloat16_rn(std * normal_of(base ^ static_cast<unsigned long long>(logical_row * hidden + col)));
    }
}

__global__ void fill_kernel(__nv_bfloat16* dst, long long n, float v) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[i] = __float2bfloat16_rn(v);
}

int blocks_for(long long n, int threads) {
    return static_cast<int>(std::min<long long>((n + threads - 1) / threads, 148LL * 32));
}

}  // namespace

void launch_init_normal(__nv_bfloat16* dst, int rows, int cols, int ld, uint64_t seed, uint64_t tensor, int64_t r0,
                        int64_t c0, int64_t C, float std, cudaStream_t s) {
    const unsigned long long base = mix(seed ^ mix(tensor * 0x9E3779B97F4A7C15ull + 17));
    init_normal_kernel<<<blocks_for(static_cast<long long>(rows) * cols, 256), 256, 0, s>>>(dst, rows, cols, ld, base,
                                                                                           r0, c0, C, std);
    CUDA_LAUNCH_CHECK();
}

void launch_init_gateup(__nv_bfloat16* dst, int ffn_local, int hidden, uint64_t seed, uint64_t gate_id, uint64_t up_id,
                        int64_t f0, float std, cudaStream_t s) {
    const unsigned long long gb = mix(seed ^ mix(gate_id * 0x9E3779B97F4A7C15ull + 17));
    const unsigned long long ub = mix(seed ^ mix(up_id * 0x9E3779B97F4A7C15ull + 17));
    init_gateup_kernel<<<blocks_for(2LL * ffn_local * hidden, 256), 256, 0, s>>>(dst, ffn_local, hidden, gb, ub, f0,
                                                                                 std);
    CUDA_LAUNCH_CHECK();
}

void launch_init_qkv(__nv_bfloat16* dst, int q_dim, int kv_dim, int hd, int hidden, uint64_t seed, uint64_t q_id,
                     uint64_t k_id, uint64_t v_id, int64_t rq0, int64_t rkv0, float std, cudaStream_t s) {
    auto base = [&](uint64_t id) { return mix(seed ^ mix(id * 0x9E3779B97F4A7C15ull + 17)); };
    const long long n = (q_dim + 2LL * kv_dim) * hidden;
    init_qkv_kernel<<<blocks_for(n, 256), 256, 0, s>>>(dst, q_dim, kv_dim, hd, hidden, base(q_id), base(k_id),
                                                       base(v_id), rq0, rkv0, std);
    CUDA_LAUNCH_CHECK();
}

__global__ void tile_weights_kernel(__nv_bfloat16* __restrict__ dst, const __nv_bfloat16* __restrict__ src, int rows,
                                    int K, int rows_p, bool untile) {
    const long long n8 = static_cast<long long>(rows_p) * K / 8;  // 16-byte groups of the tiled image
    const int KB = K / kWTileK;
    for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < n8;
         g += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e = g * 8;
        const long long tile = e / (kWTileRows * kWTileK);
        const int in = static_cast<int>(e % (kWTileRows * kWTileK));
        const int r = static_cast<int>(tile / KB) * kWTileRows + in / kWTileK;
        const long long k = (tile % KB) * kWTileK + in % kWTileK;
        if (!untile) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (r < rows) v = *reinterpret_cast<const uint4*>(src + static_cast<long long>(r) * K + k);
            *reinterpret_cast<uint4*>(dst + e) = v;
        } else if (r < rows) {
            *reinterpret_cast<uint4*>(dst + static_cast<long long>(r) * K + k) = *reinterpret_cast<const uint4*>(src + e);
        }
    }
}

void launch_tile_weights(__nv_bfloat16* dst, const __nv_bfloat16* src, int rows, int K, cudaStream_t s) {
    if (K % kWTileK) throw_invalid("tiled weights: K must be a multiple of 64");
    tile_weights_kernel<<<1184, 256, 0, s>>>(dst, src, rows, K, static_cast<int>(tiled_rows(rows)), false);
    CUDA_CHECK(cudaGetLastError());
}
void launch_untile_weights(__nv_bfloat16* dst, const __nv_bfloat16* src, int rows, int K, cudaStream_t s) {
    if (K % kWTileK) throw_invalid("tiled weights: K must be a multiple of 64");
    tile_weights_kernel<<<1184, 256, 0, s>>>(dst, src, rows, K, static_cast<int>(tiled_rows(rows)), true);
    CUDA_CHECK(cudaGetLastError());
}

void launch_fill(__nv_bfloat16* dst, int64_t n, float v, cudaStream_t s) {
    fill_kernel<<<blocks_for(n, 256), 256, 0, s>>>(dst, n, v);
    CUDA_LAUNCH_CHECK();
}

}  // namespace dbl
