// Non-GEMM verify-forward kernels (see tf_kernels.cuh).  All forward kernels are launched with PDL
// (launch.cuh): they release their dependents at entry and griddep_wait() before reading data the
// previous kernel on the stream produced.
#include <cmath>

#include "launch.cuh"
#include "sm100.cuh"
#include "tf_kernels.cuh"

namespace dbl {

namespace {

using sm100::griddep_launch_dependents;
using sm100::griddep_wait;

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

__global__ void forward_begin_kernel(LaneState* lane) {
    griddep_launch_dependents();
    griddep_wait();
    lane->start = min(lane->kv_len, lane->row0);
}
__global__ void forward_end_kernel(LaneState* lane) {
    griddep_launch_dependents();
    griddep_wait();
    lane->kv_len = lane->L + lane->c;
}

__global__ void embed_kernel(const __nv_bfloat16* __restrict__ E, int hidden, const int32_t* __restrict__ buf,
                             const LaneState* lane, float* __restrict__ resid) {
    griddep_launch_dependents();
    griddep_wait();
    const int t = blockIdx.x;
    const int start = lane->start, T = lane->L + lane->c - start;
    const int tok = t < T ? buf[start + t] : 0;
    const __nv_bfloat162* row = reinterpret_cast<const __nv_bfloat162*>(E + static_cast<long long>(tok) * hidden);
    float2* o = reinterpret_cast<float2*>(resid + static_cast<long long>(t) * hidden);
    for (int i = threadIdx.x; i < hidden / 2; i += blockDim.x) o[i] = __bfloat1622float2(row[i]);
}

// one CTA per row; every thread issues all of its (float4) loads before reducing; fixed-order
// reduction (per-thread sequential, warp xor tree, warp partials in warp order)
constexpr int kNormThreads = 256;
constexpr int kNormMaxVec = 8;  // hidden <= 256 * 4 * 8 = 8192
__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const float* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ w, int hidden,
                                                               float eps, __nv_bfloat16* __restrict__ out) {
    griddep_launch_dependents();
    __shared__ float red[kNormThreads / 32];
    const float4* row = reinterpret_cast<const float4*>(x + static_cast<long long>(blockIdx.x) * hidden);
    const int nvec = hidden / 4;
    float4 v[kNormMaxVec];
    griddep_wait();
#pragma unroll
    for (int k = 0; k < kNormMaxVec; ++k) {
        const int i = threadIdx.x + k * kNormThreads;
        v[k] = i < nvec ? row[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kNormMaxVec; ++k) {
        ss = fmaf(v[k].x, v[k].x, ss);
        ss = fmaf(v[k].y, v[k].y, ss);
        ss = fmaf(v[k].z, v[k].z, ss);
        ss = fmaf(v[k].w, v[k].w, ss);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int i = 0; i < kNormThreads / 32; ++i) tot += red[i];
    const float r = rsqrtf(tot / hidden + eps);
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(out + static_cast<long long>(blockIdx.x) * hidden);
    const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(w);
#pragma unroll
    for (int k = 0; k < kNormMaxVec; ++k) {
        const int i = threadIdx.x + k * kNormThreads;
        if (i < nvec) {
            const float2 wa = __bfloat1622float2(w2[2 * i]), wb = __bfloat1622float2(w2[2 * i + 1]);
            o[2 * i] = __floats2bfloat162_rn(v[k].x * r * wa.x, v[k].y * r * wa.y);
            o[2 * i + 1] = __floats2bfloat162_rn(v[k].z * r * wb.x, v[k].w * r * wb.y);
        }
    }
}

__device__ __forceinline__ __nv_bfloat16* kv_addr(__nv_bfloat16* base, const int32_t* pt, int n_kv, int hd, int h,
                                                  int pos) {
    const int phys = pt[pos / kPage];
    return base + ((static_cast<long long>(phys) * n_kv + h) * kPage + (pos % kPage)) * hd;
}

// one warp per (token, head slot): slots [0, nh) q heads, [nh, nh+nkv) k heads, [nh+nkv, nh+2nkv) v heads
template <int HD>
__global__ void qkv_post_kernel(const __nv_bfloat16* __restrict__ qkv, int nh, int nkv, const __nv_bfloat16* qn,
                                const __nv_bfloat16* kn, float eps, float theta, const LaneState* lane, KVView kv,
                                __nv_bfloat16* __restrict__ qbuf) {
    griddep_launch_dependents();
    griddep_wait();
    constexpr int E = HD / 32;  // elements per lane: dims lane + 32*e
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, ln = threadIdx.x & 31;
    const int slots = nh + 2 * nkv;
    const int t = warp / slots, slot = warp % slots;
    const int start = lane->start, T = lane->L + lane->c - start;
    if (t >= T) return;
    const int pos = start + t;
    const __nv_bfloat16* src = qkv + static_cast<long long>(t) * slots * HD + static_cast<long long>(slot) * HD;
    float x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = __bfloat162float(src[ln + 32 * e]);
    const bool is_q = slot < nh, is_k = !is_q && slot < nh + nkv;
    if (is_q || is_k) {
        const __nv_bfloat16* nw = is_q ? qn : kn;
        if (nw) {  // per-head RMSNorm (Qwen3 q_norm / k_norm)
            float ss = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) ss = fmaf(x[e], x[e], ss);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
            const float r = rsqrtf(ss / HD + eps);
#pragma unroll
            for (int e = 0; e < E; ++e) x[e] = __bfloat162float(__float2bfloat16_rn(x[e] * r * __bfloat162float(nw[ln + 32 * e])));
        }
        // RoPE (rotate-half): dim d < HD/2 pairs with d + HD/2 — same lane, element e and e + E/2
        float y[E];
#pragma unroll
        for (int e = 0; e < E / 2; ++e) {
            const int d = ln + 32 * e;
            const float inv = powf(theta, -2.0f * static_cast<float>(d) / static_cast<float>(HD));
            float sn, cs;
            sincosf(static_cast<float>(pos) * inv, &sn, &cs);
            y[e] = x[e] * cs - x[e + E / 2] * sn;
            y[e + E / 2] = x[e + E / 2] * cs + x[e] * sn;
        }
        if (is_q) {
            __nv_bfloat16* dq = qbuf + (static_cast<long long>(t) * nh + slot) * HD;
#pragma unroll
            for (int e = 0; e < E; ++e) dq[ln + 32 * e] = __float2bfloat16_rn(y[e]);
        } else {
            __nv_bfloat16* dk = kv_addr(kv.k, kv.page_table, nkv, HD, slot - nh, pos);
#pragma unroll
            for (int e = 0; e < E; ++e) dk[ln + 32 * e] = __float2bfloat16_rn(y[e]);
        }
    } else {
        __nv_bfloat16* dv = kv_addr(kv.v, kv.page_table, nkv, HD, slot - nh - nkv, pos);
#pragma unroll
        for (int e = 0; e < E; ++e) dv[ln + 32 * e] = __float2bfloat16_rn(x[e]);
    }
}

constexpr int kQTile = 16;
constexpr int kAttnThreads = 256;
constexpr int kAttnWarps = kAttnThreads / 32;

// grid (n_kv, key chunks of kAttnChunk, token tiles of kQTile).  One CTA stages its chunk's K (padded
// rows, conflict-free bf16x2 reads) and V in shared memory; each warp takes (token, q head) pairs:
// lanes score keys lane, lane+32 (sequential dot product), warp max / sum, then lanes accumulate their
// hd/32 output dims over the chunk's keys in order.  Partial (m, l, o) per (token, head, chunk).
template <int HD>
__global__ void __launch_bounds__(kAttnThreads) attn_chunk_kernel(const __nv_bfloat16* __restrict__ qbuf, int nh,
                                                                  int nkv, KVView kv, const LaneState* lane,
                                                                  int max_chunks, float* __restrict__ part_o,
                                                                  float* __restrict__ part_ml) {
    griddep_launch_dependents();
    constexpr int KS = HD + 2;
    constexpr int NK = kAttnChunk;
    __shared__ __align__(16) __nv_bfloat16 sK[NK * KS];
    __shared__ __align__(16) __nv_bfloat16 sV[NK * HD];
    __shared__ float sP[kAttnWarps][NK];
    __shared__ float sQ[kAttnWarps][HD];
    griddep_wait();
    const int h = blockIdx.x, j = blockIdx.y, qt = blockIdx.z;
    const int start = lane->start, T = lane->L + lane->c - start;
    const int t0 = qt * kQTile, t1 = min(T, t0 + kQTile);
    if (t0 >= t1) return;
    const int pmax = start + t1 - 1;
    const int k0 = j * NK;
    if (k0 > pmax) return;
    const int nk = min(NK, pmax - k0 + 1);
    // chunk = one KV page (kAttnChunk == kPage): contiguous [nk][HD] rows for this head
    const __nv_bfloat16* kp = kv_addr(kv.k, kv.page_table, nkv, HD, h, k0);
    const __nv_bfloat16* vp = kv_addr(kv.v, kv.page_table, nkv, HD, h, k0);
    for (int idx = threadIdx.x; idx < nk * (HD / 8); idx += kAttnThreads) {
        const int i = idx / (HD / 8), c8 = idx % (HD / 8);
        const uint4 kk = reinterpret_cast<const uint4*>(kp + i * HD)[c8];
        const uint4 vv = reinterpret_cast<const uint4*>(vp + i * HD)[c8];
        const uint32_t* kw = reinterpret_cast<const uint32_t*>(&kk);
        uint32_t* dk = reinterpret_cast<uint32_t*>(sK + i * KS + c8 * 8);  // 4-byte aligned (KS even)
        dk[0] = kw[0]; dk[1] = kw[1]; dk[2] = kw[2]; dk[3] = kw[3];
        reinterpret_cast<uint4*>(sV + i * HD)[c8] = vv;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const int g = nh / nkv;
    const float scale = rsqrtf(static_cast<float>(HD));
    float* p = sP[warp];
    float* q = sQ[warp];
    for (int pair = warp; pair < (t1 - t0) * g; pair += kAttnWarps) {
        const int t = t0 + pair / g, hq = h * g + pair % g;
        const int pos = start + t;
        if (pos < k0) continue;
        const int n = min(nk, pos - k0 + 1);
        const __nv_bfloat16* qs = qbuf + (static_cast<long long>(t) * nh + hq) * HD;
        for (int d = ln; d < HD; d += 32) q[d] = __bfloat162float(qs[d]);
        __syncwarp();
        float s0 = -INFINITY, s1 = -INFINITY;
        if (ln < n) {
            const __nv_bfloat162* kr = reinterpret_cast<const __nv_bfloat162*>(sK + ln * KS);
            float s = 0.f;
#pragma unroll 16
            for (int d2 = 0; d2 < HD / 2; ++d2) {
                const float2 kf = __bfloat1622float2(kr[d2]);
                s = fmaf(q[2 * d2], kf.x, s);
                s = fmaf(q[2 * d2 + 1], kf.y, s);
            }
            s0 = s * scale;
        }
        if (ln + 32 < n) {
            const __nv_bfloat162* kr = reinterpret_cast<const __nv_bfloat162*>(sK + (ln + 32) * KS);
            float s = 0.f;
#pragma unroll 16
            for (int d2 = 0; d2 < HD / 2; ++d2) {
                const float2 kf = __bfloat1622float2(kr[d2]);
                s = fmaf(q[2 * d2], kf.x, s);
                s = fmaf(q[2 * d2 + 1], kf.y, s);
            }
            s1 = s * scale;
        }
        float mx = fmaxf(s0, s1);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const float e0 = ln < n ? __expf(s0 - mx) : 0.f, e1 = ln + 32 < n ? __expf(s1 - mx) : 0.f;
        p[ln] = e0;
        p[ln + 32] = e1;
        float l = e0 + e1;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
        __syncwarp();
        float o[HD / 32];
#pragma unroll
        for (int k = 0; k < HD / 32; ++k) o[k] = 0.f;
        for (int i = 0; i < n; ++i) {
            const float pi = p[i];
#pragma unroll
            for (int k = 0; k < HD / 32; ++k) o[k] = fmaf(pi, __bfloat162float(sV[i * HD + ln + 32 * k]), o[k]);
        }
        const long long slot = (static_cast<long long>(t) * nh + hq) * max_chunks + j;
#pragma unroll
        for (int k = 0; k < HD / 32; ++k) part_o[slot * HD + ln + 32 * k] = o[k];
        if (ln == 0) {
            part_ml[2 * slot] = mx;
            part_ml[2 * slot + 1] = l;
        }
        __syncwarp();
    }
}

// one warp per (token, q head): combine the position's chunks in chunk order
template <int HD>
__global__ void attn_combine_kernel(int nh, int max_chunks, const LaneState* lane, const float* __restrict__ part_o,
                                    const float* __restrict__ part_ml, __nv_bfloat16* __restrict__ out) {
    griddep_launch_dependents();
    griddep_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, ln = threadIdx.x & 31;
    const int start = lane->start, T = lane->L + lane->c - start;
    const int t = warp / nh, hq = warp % nh;
    if (t >= T) return;
    const int pos = start + t;
    const int nch = pos / kAttnChunk + 1;
    const long long base = (static_cast<long long>(t) * nh + hq) * max_chunks;
    float M = -INFINITY;
    for (int j = 0; j < nch; ++j) M = fmaxf(M, part_ml[2 * (base + j)]);
    float den = 0.f, acc[HD / 32];
#pragma unroll
    for (int k = 0; k < HD / 32; ++k) acc[k] = 0.f;
    for (int j = 0; j < nch; ++j) {
        const float w = __expf(part_ml[2 * (base + j)] - M);
        den = fmaf(part_ml[2 * (base + j) + 1], w, den);
#pragma unroll
        for (int k = 0; k < HD / 32; ++k) acc[k] = fmaf(part_o[(base + j) * HD + ln + 32 * k], w, acc[k]);
    }
    const float inv = 1.0f / den;
#pragma unroll
    for (int k = 0; k < HD / 32; ++k)
        out[static_cast<long long>(t) * nh * HD + hq * HD + ln + 32 * k] = __float2bfloat16_rn(acc[k] * inv);
}

int blocks_for(long long n, int threads) {
    return static_cast<int>(std::min<long long>((n + threads - 1) / threads, 148LL * 32));
}

}  // namespace

void launch_embed(const __nv_bfloat16* E, int hidden, const int32_t* buf, const LaneState* lane, int tp, float* resid,
                  cudaStream_t s) {
    launch_pdl(embed_kernel, dim3(tp), dim3(256), 0, s, E, hidden, buf, lane, resid);
}

void launch_rmsnorm(const float* x, const __nv_bfloat16* w, int hidden, float eps, int tp, __nv_bfloat16* out,
                    cudaStream_t s) {
    if (hidden % 4 || hidden > kNormThreads * 4 * kNormMaxVec) throw_invalid("rmsnorm: hidden unsupported");
    launch_pdl(rmsnorm_kernel, dim3(tp), dim3(kNormThreads), 0, s, x, w, hidden, eps, out);
}

void launch_qkv_post(const __nv_bfloat16* qkv, int nh, int nkv, int hd, const __nv_bfloat16* qn,
                     const __nv_bfloat16* kn, float eps, float theta, const LaneState* lane, KVView kv,
                     __nv_bfloat16* qbuf, int tp, cudaStream_t s) {
    const long long warps = static_cast<long long>(tp) * (nh + 2 * nkv);
    const int blocks = static_cast<int>((warps * 32 + 255) / 256);
    if (hd == 128)
        launch_pdl(qkv_post_kernel<128>, dim3(blocks), dim3(256), 0, s, qkv, nh, nkv, qn, kn, eps, theta, lane, kv, qbuf);
    else if (hd == 64)
        launch_pdl(qkv_post_kernel<64>, dim3(blocks), dim3(256), 0, s, qkv, nh, nkv, qn, kn, eps, theta, lane, kv, qbuf);
    else
        throw_invalid("head_dim must be 64 or 128");
}

void launch_attention(const __nv_bfloat16* qbuf, int nh, int nkv, int hd, KVView kv, const LaneState* lane, int tp,
                      int max_chunks, float* part_o, float* part_ml, __nv_bfloat16* out, cudaStream_t s) {
    static_assert(kAttnChunk == kPage, "attention chunk must be one KV page");
    const dim3 grid(nkv, max_chunks, (tp + kQTile - 1) / kQTile);
    const int cblocks = (tp * nh * 32 + 255) / 256;
    if (hd == 128) {
        launch_pdl(attn_chunk_kernel<128>, grid, dim3(kAttnThreads), 0, s, qbuf, nh, nkv, kv, lane, max_chunks, part_o,
                   part_ml);
        launch_pdl(attn_combine_kernel<128>, dim3(cblocks), dim3(256), 0, s, nh, max_chunks, lane,
                   static_cast<const float*>(part_o), static_cast<const float*>(part_ml), out);
    } else if (hd == 64) {
        launch_pdl(attn_chunk_kernel<64>, grid, dim3(kAttnThreads), 0, s, qbuf, nh, nkv, kv, lane, max_chunks, part_o,
                   part_ml);
        launch_pdl(attn_combine_kernel<64>, dim3(cblocks), dim3(256), 0, s, nh, max_chunks, lane,
                   static_cast<const float*>(part_o), static_cast<const float*>(part_ml), out);
    } else {
        throw_invalid("head_dim must be 64 or 128");
    }
}

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

void launch_forward_begin(LaneState* lane, cudaStream_t s) { launch_pdl(forward_begin_kernel, dim3(1), dim3(1), 0, s, lane); }
void launch_forward_end(LaneState* lane, cudaStream_t s) { launch_pdl(forward_end_kernel, dim3(1), dim3(1), 0, s, lane); }

}  // namespace dbl
