// Retrieval kernels (K1 lookup, K1b insert) and the DeviceStore host object.
// Semantics: HierarchicalDatastore::lookup / NGramIndex::insert (datastore.cpp:9-132).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "store.cuh"

namespace dbl {

namespace {

// 64-bit hash of an n-gram given newest-first (k_0 = its last token): the index key.  Bit 63 is
// clear and 0 is never produced, so 0 marks an empty table slot and ~0 an invalid entry.
constexpr unsigned long long kNoKey = ~0ull;
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned long long ngram_step(unsigned long long h, int tok) {
    return mix64(h ^ (static_cast<unsigned long long>(static_cast<uint32_t>(tok)) * 0x9E3779B97F4A7C15ull));
}
__host__ __device__ __forceinline__ unsigned long long ngram_key(unsigned long long h, int n) {
    unsigned long long k = mix64(h + static_cast<unsigned long long>(n) * 0xD6E8FEB86659FD93ull) & 0x7FFFFFFFFFFFFFFFull;
    return k ? k : 1ull;
}
constexpr unsigned long long kHashSeed = 0x243F6A8885A308D3ull;

constexpr int kLookupThreads = 512;
constexpr int kWarps = kLookupThreads / 32;

// 128-bit lexicographic key of an occurrence: (step, avail, seq_id, end_pos), datastore.cpp:60-65.
// hi = step with the sign bit flipped (signed -> unsigned order); lo = avail<<48 | seq<<24 | end.
// lo == 0 <=> "no occurrence" (a valid occurrence has avail >= 1).
struct Key {
    unsigned long long hi, lo;
};
__device__ __forceinline__ bool key_gt(const Key& a, const Key& b) {
    return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo);
}
__device__ __forceinline__ Key key_shfl_max(Key k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Key o;
        o.hi = __shfl_xor_sync(0xffffffffu, k.hi, off);
        o.lo = __shfl_xor_sync(0xffffffffu, k.lo, off);
        if (key_gt(o, k)) k = o;
    }
    return k;
}

struct LookupOut {
    int n, src, order;
};

// One CTA answers one lookup.  ctx[0, L) is the query; candidates are written to out[0, n).
// Shared-memory staging: the context suffix (probe key, reversed) and per-(layer, order) winners.
__device__ void lookup_cta(const StoreDesc* __restrict__ sd, const int32_t* __restrict__ ctx, int L,
                           int d, int32_t* __restrict__ out, LookupOut* res) {
    __shared__ int32_t s_key[kMaxOrder];   // s_key[j] = ctx[L-1-j]
    __shared__ Key s_best[3][kMaxOrder + 1];
    __shared__ int s_pld[kWarps];
    __shared__ int s_pld_end[kMaxOrder + 1];
    __shared__ int s_choice[4];  // src, order, from, layer-seq
    __shared__ uint2 s_run[3][kMaxOrder + 1];  // index probes: (run start, length) per (layer, order)
    __shared__ Key s_red3[3][kWarps];
    __shared__ Key s_redn[kMaxOrder][kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = sd->max_order;
    const int nkey = min(N, L);
    if (tid < kMaxOrder) s_key[tid] = tid < nkey ? ctx[L - 1 - tid] : -1;
    __syncthreads();

    // ---- index probes, all in flight together: thread l * kMaxOrder + n - 1 hashes the context's
    // order-n suffix and probes layer l's table (one 16-byte load per slot)
    {
        const int l = tid / kMaxOrder, n = tid % kMaxOrder + 1;
        if (l < 3) {
            const LayerDesc& ly = sd->layer[l];
            uint2 run = make_uint2(0u, 0u);
            if (ly.idx_tokens > 0 && (l != 2 || sd->rejected_enabled) && n <= nkey &&
                n <= min(ly.max_order, ly.idx_order)) {
                unsigned long long hk = kHashSeed;
                for (int j = 0; j < n; ++j) hk = ngram_step(hk, s_key[j]);
                hk = ngram_key(hk, n);
                for (unsigned slot = static_cast<unsigned>(hk) & ly.idx_mask;; slot = (slot + 1) & ly.idx_mask) {
                    const uint4 e = __ldg(reinterpret_cast<const uint4*>(ly.idx_table + slot));
                    const unsigned long long k = (static_cast<unsigned long long>(e.y) << 32) | e.x;
                    if (k == 0ull) break;
                    if (k == hk) {
                        run = make_uint2(e.z, e.w);
                        break;
                    }
                }
            }
            s_run[l][n] = run;
        }
    }

    // ---- unindexed tails [idx_tokens, n_tokens) (the dynamic / rejected layers): the best occurrence
    // per order n, all orders in one pass; a candidate's loads (its n-gram, its sequence record) are
    // issued together
    for (int l = 0; l < 3; ++l) {
        const LayerDesc ly = sd->layer[l];
        const bool enabled = (l != 2 || sd->rejected_enabled) && ly.n_tokens > ly.idx_tokens;
        const int Nl = min(nkey, ly.max_order);
        if (!enabled || Nl < 1) {  // uniform: nothing to scan, no reduction
            if (tid <= kMaxOrder) s_best[l][tid] = Key{0ull, 0ull};
            continue;
        }
        Key best[kMaxOrder + 1];
#pragma unroll
        for (int n = 0; n <= kMaxOrder; ++n) best[n] = Key{0ull, 0ull};
        const int k0 = s_key[0];
        for (int p = ly.idx_tokens + tid; p < ly.n_tokens; p += kLookupThreads) {
            if (__ldg(ly.tokens + p) != k0) continue;  // cheap filter: last token must match
            const int q = __ldg(ly.seq_of + p);
            int tk[kMaxOrder];
#pragma unroll
            for (int j = 1; j < kMaxOrder; ++j) tk[j] = (j < Nl && p - j >= 0) ? __ldg(ly.tokens + p - j) : -1;
            const int st = __ldg(ly.seq_start + q);
            const int len = __ldg(ly.seq_len + q);
            const long long stp = __ldg(ly.seq_step + q);
            const int e = p - st;
            const int avail = min(len - e - 1, d);
            if (avail <= 0) continue;
            const int mmax = min(Nl, e + 1);
            int m = 1;
#pragma unroll
            for (int j = 1; j < kMaxOrder; ++j)
                if (m == j && j < mmax && tk[j] == s_key[j]) m = j + 1;
            Key k;
            k.hi = static_cast<unsigned long long>(stp) ^ 0x8000000000000000ull;
            k.lo = (static_cast<unsigned long long>(avail) << 48) |
                   (static_cast<unsigned long long>(q) << 24) | static_cast<unsigned long long>(e);
#pragma unroll
            for (int n = 1; n <= kMaxOrder; ++n)
                if (n <= m && key_gt(k, best[n])) best[n] = k;
        }
        // block max-reduce, every order at once: warp maxima -> shared, then warp n - 1 reduces order n
#pragma unroll
        for (int n = 1; n <= kMaxOrder; ++n) {
            const Key k = key_shfl_max(best[n]);
            if (lane == 0 && n <= N) s_redn[n - 1][warp] = k;
        }
        __syncthreads();
        if (warp < N) {
            Key r = lane < kWarps ? s_redn[warp][lane] : Key{0ull, 0ull};
            r = key_shfl_max(r);
            if (lane == 0) s_best[l][warp + 1] = r;
        }
        __syncthreads();
    }
    __syncthreads();  // s_run, and s_best of skipped layers

    // ---- indexed runs, from the highest order down: merge each layer's run into its best occurrence
    // at that order; stop at the first order where any layer has one (the choice below never looks at
    // lower orders then).  Hash collisions are rejected by comparing the n-gram's tokens.
    for (int n = nkey; n >= 1; --n) {
        if (s_run[0][n].y + s_run[1][n].y + s_run[2][n].y > 0u) {  // uniform
            Key bl[3] = {{0ull, 0ull}, {0ull, 0ull}, {0ull, 0ull}};
#pragma unroll
            for (int l = 0; l < 3; ++l) {
                const LayerDesc& ly = sd->layer[l];
                const uint2 run = s_run[l][n];
                for (int i = tid; i < static_cast<int>(run.y); i += kLookupThreads) {
                    const unsigned long long oc = __ldg(ly.idx_occ + run.x + i);
                    const int p = static_cast<int>(oc & 0xFFFFFFFFull), q = static_cast<int>(oc >> 32);
                    int tk[kMaxOrder];
#pragma unroll
                    for (int j = 0; j < kMaxOrder; ++j) tk[j] = j < n ? __ldg(ly.tokens + p - j) : 0;
                    const int st = __ldg(ly.seq_start + q);
                    const int len = __ldg(ly.seq_len + q);
                    const long long stp = __ldg(ly.seq_step + q);
                    bool match = true;
#pragma unroll
                    for (int j = 0; j < kMaxOrder; ++j) match &= j >= n || tk[j] == s_key[j];
                    const int e = p - st;
                    const int avail = min(len - e - 1, d);
                    if (!match || avail <= 0) continue;
                    Key k;
                    k.hi = static_cast<unsigned long long>(stp) ^ 0x8000000000000000ull;
                    k.lo = (static_cast<unsigned long long>(avail) << 48) |
                           (static_cast<unsigned long long>(q) << 24) | static_cast<unsigned long long>(e);
                    if (key_gt(k, bl[l])) bl[l] = k;
                }
            }
#pragma unroll
            for (int l = 0; l < 3; ++l) {
                const Key k = key_shfl_max(bl[l]);
                if (lane == 0) s_red3[l][warp] = k;
            }
            __syncthreads();
            if (warp < 3) {
                Key r = lane < kWarps ? s_red3[warp][lane] : Key{0ull, 0ull};
                r = key_shfl_max(r);
                if (lane == 0 && key_gt(r, s_best[warp][n])) s_best[warp][n] = r;
            }
            __syncthreads();
        }
        bool hit = false;
        for (int l = 0; l < 3; ++l)
            if ((l != 2 || sd->rejected_enabled) && s_best[l][n].lo != 0ull) hit = true;
        if (hit) break;
    }

    // ---- choose: order desc, then prior > dynamic > rejected (datastore.cpp:88-107)
    if (tid == 0) {
        s_choice[0] = DBL_SRC_MISS;
        for (int n = nkey; n >= 1 && s_choice[0] == DBL_SRC_MISS; --n) {
            for (int l = 0; l < 3; ++l) {
                if (l == 2 && !sd->rejected_enabled) continue;
                if (s_best[l][n].lo != 0ull) {
                    s_choice[0] = l;
                    s_choice[1] = n;
                    s_choice[2] = static_cast<int>((s_best[l][n].lo >> 24) & 0xFFFFFFull);  // seq
                    s_choice[3] = static_cast<int>(s_best[l][n].lo & 0xFFFFFFull);          // end
                    break;
                }
            }
        }
    }
    __syncthreads();
    if (s_choice[0] != DBL_SRC_MISS) {
        const LayerDesc ly = sd->layer[s_choice[0]];
        const int q = s_choice[2], e = s_choice[3];
        const int st = ly.seq_start[q], len = ly.seq_len[q];
        const int from = e + 1, to = min(from + d, len);  // continuation, datastore.cpp:73-78
        for (int i = tid; i < to - from; i += kLookupThreads) out[i] = ly.tokens[st + from + i];
        if (tid == 0) *res = LookupOut{to - from, s_choice[0], s_choice[1]};
        return;
    }

    // ---- PLD fallback (datastore.cpp:109-128): longest n first, then the latest earlier end
    const int nf = min(N, L - 1);
    int maxend[kMaxOrder + 1];
#pragma unroll
    for (int n = 0; n <= kMaxOrder; ++n) maxend[n] = -1;
    if (nf >= 1) {
        for (int end = tid; end <= L - 2; end += kLookupThreads) {
            if (ctx[end] != s_key[0]) continue;
            int m = 1;
            const int mmax = min(nf, end + 1);
            while (m < mmax && ctx[end - m] == s_key[m]) ++m;
#pragma unroll
            for (int n = 1; n <= kMaxOrder; ++n)
                if (n <= m) maxend[n] = max(maxend[n], end);
        }
    }
    for (int n = 1; n <= kMaxOrder; ++n) {
        if (n > N) break;
        int v = maxend[n];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) s_pld[warp] = v;
        __syncthreads();
        if (warp == 0) {
            int r = lane < kWarps ? s_pld[lane] : -1;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) r = max(r, __shfl_xor_sync(0xffffffffu, r, off));
            if (lane == 0) s_pld_end[n] = r;
        }
        __syncthreads();
    }
    if (tid == 0) {
        s_choice[0] = DBL_SRC_MISS;
        for (int n = nf; n >= 1; --n) {
            if (s_pld_end[n] >= 0) {
                s_choice[0] = DBL_SRC_CONTEXT;
                s_choice[1] = n;
                s_choice[2] = s_pld_end[n] + 1;
                break;
            }
        }
    }
    __syncthreads();
    if (s_choice[0] == DBL_SRC_CONTEXT) {
        const int from = s_choice[2], to = min(from + d, L);
        for (int i = tid; i < to - from; i += kLookupThreads) out[i] = ctx[from + i];
        if (tid == 0) *res = LookupOut{max(to - from, 0), DBL_SRC_CONTEXT, s_choice[1]};
    } else if (tid == 0) {
        *res = LookupOut{0, DBL_SRC_MISS, 0};
    }
}

__device__ __forceinline__ void count_stat(StoreDesc* sd, int src) {
    atomicAdd(&sd->stats[0], 1ull);
    atomicAdd(&sd->stats[1 + (src == DBL_SRC_CONTEXT ? 3 : src == DBL_SRC_MISS ? 4 : src)], 1ull);
}

__global__ void __launch_bounds__(kLookupThreads) lookup_lane_kernel(StoreDesc* sd, int32_t* buf,
                                                                     LaneState* lane, int d) {
    __shared__ LookupOut res;
    const int L = lane->L;
    lookup_cta(sd, buf, L, d, buf + L, &res);
    __syncthreads();
    if (threadIdx.x == 0) {
        lane->c = res.n;
        lane->src = res.src;
        lane->order = res.order;
        count_stat(sd, res.src);
    }
}

__global__ void __launch_bounds__(kLookupThreads) lookup_batch_kernel(
    StoreDesc* sd, const int64_t* __restrict__ offsets, const int32_t* __restrict__ toks,
    const int32_t* __restrict__ depths, int d_cap, int32_t* out_cands, int32_t* out_n,
    int32_t* out_src, int32_t* out_order) {
    __shared__ LookupOut res;
    const int q = blockIdx.x;
    const int64_t a = offsets[q], b = offsets[q + 1];
    lookup_cta(sd, toks + a, static_cast<int>(b - a), depths[q], out_cands + static_cast<int64_t>(q) * d_cap, &res);
    __syncthreads();
    if (threadIdx.x == 0) {
        out_n[q] = res.n;
        out_src[q] = res.src;
        out_order[q] = res.order;
        count_stat(sd, res.src);
    }
}

// K1b: append one sequence to a layer (NGramIndex::insert, datastore.cpp:9-20)
__global__ void append_kernel(StoreDesc* sd, int layer, const int32_t* __restrict__ src, int n,
                              long long step) {
    LayerDesc& ly = sd->layer[layer];
    const int nt = ly.n_tokens, ns = ly.n_seqs;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        ly.tokens[nt + i] = src[i];
        ly.seq_of[nt + i] = ns;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ly.seq_start[ns] = nt;
        ly.seq_len[ns] = n;
        ly.seq_step[ns] = step;
        ly.n_tokens = nt + n;
        ly.n_seqs = ns + 1;
    }
}

__global__ void set_layer_kernel(StoreDesc* sd, int layer, LayerDesc v, int keep_counts) {
    LayerDesc& ly = sd->layer[layer];
    const int nt = ly.n_tokens, ns = ly.n_seqs;
    ly = v;
    if (keep_counts) { ly.n_tokens = nt; ly.n_seqs = ns; }
}
// bulk layer load (build_prior): sequence s owns tokens [start[s], start[s] + len[s])
__global__ void fill_seq_of_kernel(int32_t* seq_of, const int32_t* __restrict__ start, const int32_t* __restrict__ len,
                                   int n_seqs) {
    for (int q = blockIdx.x; q < n_seqs; q += gridDim.x) {
        const int a = start[q], n = len[q];
        for (int i = threadIdx.x; i < n; i += blockDim.x) seq_of[a + i] = q;
    }
}
__global__ void add_stats_kernel(StoreDesc* sd, long long d0, long long d1, long long d2, long long d3,
                                 long long d4, long long d5) {
    const long long d[6] = {d0, d1, d2, d3, d4, d5};
    if (threadIdx.x < 6) sd->stats[threadIdx.x] += static_cast<unsigned long long>(d[threadIdx.x]);
}
__global__ void set_store_kernel(StoreDesc* sd, int max_order, int rej) {
    sd->max_order = max_order;
    sd->rejected_enabled = rej;
}

// n-gram index build: one (key, position) entry per (position p, order n) whose n-gram lies inside p's
// sequence and whose sequence continues after p (an occurrence with nothing after it is never
// returned: avail = min(remaining, d) <= 0, datastore.cpp:57-58); others get kNoKey (sorted last)
__global__ void index_entries_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ seq_of,
                                     const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_len,
                                     int nt, int N, unsigned long long* keys, unsigned long long* vals) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nt; p += gridDim.x * blockDim.x) {
        const int q = seq_of[p];
        const int e = p - seq_start[q];
        const bool cont = seq_len[q] - e - 1 >= 1;
        unsigned long long h = kHashSeed;
        for (int n = 1; n <= N; ++n) {
            const bool ok = cont && e >= n - 1;
            if (ok) h = ngram_step(h, tokens[p - n + 1]);
            keys[static_cast<long long>(p) * N + n - 1] = ok ? ngram_key(h, n) : kNoKey;
            vals[static_cast<long long>(p) * N + n - 1] =
                (static_cast<unsigned long long>(q) << 32) | static_cast<uint32_t>(p);
        }
    }
}
// run r of the sorted entries -> its table slot (linear probing; keys are unique)
__global__ void index_table_kernel(const unsigned long long* __restrict__ ukeys, const uint32_t* __restrict__ start,
                                   const uint32_t* __restrict__ count, const int* __restrict__ n_runs,
                                   IdxSlot* table, uint32_t mask) {
    const int R = *n_runs;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
        const unsigned long long k = ukeys[r];
        if (k == kNoKey) continue;  // the run of invalid entries
        unsigned slot = static_cast<unsigned>(k) & mask;
        while (atomicCAS(&table[slot].key, 0ull, k) != 0ull) slot = (slot + 1) & mask;
        table[slot].start = start[r];
        table[slot].count = count[r];
    }
}

}  // namespace

LayerDesc DeviceStore::desc_of(const HostLayer& h) const {
    LayerDesc v{};
    v.tokens = h.tokens.p;
    v.seq_of = h.seq_of.p;
    v.seq_start = h.seq_start.p;
    v.seq_len = h.seq_len.p;
    v.seq_step = h.seq_step.p;
    v.n_tokens = h.n_tokens;
    v.n_seqs = h.n_seqs;
    v.max_order = h.max_order;
    v.idx_tokens = h.idx_tokens;
    v.idx_table = h.idx_table.p;
    v.idx_occ = h.idx_occ.p;
    v.idx_mask = h.idx_mask;
    v.idx_order = h.idx_order;
    return v;
}

// Index the layer's current tokens (all orders 1..max_order): entries -> radix sort by key -> run-length
// encode -> exclusive scan (run starts) -> open-addressing table of >= 2x the distinct n-grams.  The
// layer's tokens / seq_of / seq_start / seq_len must be complete on stream s.
void DeviceStore::build_index(int l, cudaStream_t s) {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    DeviceGuard g(device_);
    HostLayer& h = layers_[l];
    h.idx_tokens = 0;
    const int nt = h.n_tokens, N = h.max_order;
    if (nt <= 0) {
        LayerDesc v = desc_of(h);
        set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 1);
        CUDA_LAUNCH_CHECK();
        return;
    }
    const long long E = static_cast<long long>(nt) * N;
    if (E >= (1LL << 31)) throw_runtime("datastore index exceeds 2^31 entries");
    const int En = static_cast<int>(E);
    DevBuf<unsigned long long> k_in(En), k_out(En), ukeys(En), v_in(En);
    h.idx_occ.alloc(En);
    DevBuf<uint32_t> cnt(En), st(En);
    DevBuf<int> n_runs(1);
    index_entries_kernel<<<std::min((nt + 255) / 256, 4096), 256, 0, s>>>(h.tokens.p, h.seq_of.p, h.seq_start.p,
                                                                            h.seq_len.p, nt, N, k_in.p, v_in.p);
    CUDA_LAUNCH_CHECK();
    size_t b1 = 0, b2 = 0, b3 = 0;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, b1, k_in.p, k_out.p, v_in.p, h.idx_occ.p, En, 0, 64, s));
    CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(nullptr, b2, k_out.p, ukeys.p, cnt.p, n_runs.p, En, s));
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, b3, cnt.p, st.p, En, s));
    DevBuf<uint8_t> tmp(std::max({b1, b2, b3, size_t(1)}));
    size_t tb = tmp.n;
    CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k_in.p, k_out.p, v_in.p, h.idx_occ.p, En, 0, 64, s));
    tb = tmp.n;
    CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(tmp.p, tb, k_out.p, ukeys.p, cnt.p, n_runs.p, En, s));
    int R = 0;
    CUDA_CHECK(cudaMemcpyAsync(&R, n_runs.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    tb = tmp.n;
    CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, st.p, R, s));
    uint32_t cap = 1024;
    while (cap < 2u * static_cast<uint32_t>(R)) cap <<= 1;
    h.idx_table.alloc(cap);
    h.idx_table.zero(s);
    index_table_kernel<<<std::min((R + 255) / 256 + 1, 4096), 256, 0, s>>>(ukeys.p, st.p, cnt.p, n_runs.p,
                                                                           h.idx_table.p, cap - 1);
    CUDA_LAUNCH_CHECK();
    h.idx_mask = cap - 1;
    h.idx_order = N;
    h.idx_tokens = nt;
    LayerDesc v = desc_of(h);
    set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 1);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaStreamSynchronize(s));  // the temporaries above are freed on return
}

int64_t DeviceStore::index_entries(int l) const {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    return layers_[l].idx_tokens > 0 ? static_cast<int64_t>(layers_[l].idx_occ.n) : 0;
}

DeviceStore::DeviceStore(int max_order, int depth, int device)
    : device_(device), max_order_(max_order), depth_(depth) {
    if (max_order < 1 || max_order > kMaxOrder)
        throw_invalid("datastore max_order must be in [1, " + std::to_string(kMaxOrder) + "]");
    require_device(device);
    DeviceGuard g(device);
    CUDA_CHECK(cudaMalloc(&desc_dev_, sizeof(StoreDesc)));
    CUDA_CHECK(cudaMemset(desc_dev_, 0, sizeof(StoreDesc)));
    for (Staging& r : staging_) r.buf.alloc(1 << 16);  // grown on demand (insert)
    for (int l = 0; l < 3; ++l) {
        layers_[l].max_order = max_order;
        grow(l, 1024, 64, 0);
    }
    set_store_kernel<<<1, 1>>>(desc_dev_, max_order_, 1);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaDeviceSynchronize());
}

DeviceStore::~DeviceStore() {
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    if (desc_dev_) cudaFree(desc_dev_);
    for (Staging& r : staging_)
        for (auto& e : r.pend) cudaEventDestroy(e.second);
}

// Insert payloads go through two mapped pinned rings used alternately.  Switching to a ring waits (on
// the host, per stream that appended from it) only for that ring's own earlier append kernels — not
// for the device: a wrap never stalls the decode loop's other streams.
void DeviceStore::Staging::drain() {
    for (auto& e : pend) CUDA_CHECK(cudaEventSynchronize(e.second));
}
void DeviceStore::Staging::mark(cudaStream_t s) {
    for (auto& e : pend)
        if (e.first == s) {
            CUDA_CHECK(cudaEventRecord(e.second, s));
            return;
        }
    cudaEvent_t ev;
    CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(ev, s));
    pend.emplace_back(s, ev);
}

void DeviceStore::push_desc(cudaStream_t) {}

void DeviceStore::grow(int l, int need_tok, int need_seq, cudaStream_t s) {
    HostLayer& h = layers_[l];
    bool changed = false;
    if (need_tok > h.tok_cap) {
        int cap = std::max(need_tok, std::max(1024, h.tok_cap * 2));
        DevBuf<int32_t> t(cap), so(cap);
        if (h.n_tokens) {
            CUDA_CHECK(cudaMemcpyAsync(t.p, h.tokens.p, h.n_tokens * 4, cudaMemcpyDeviceToDevice, s));
            CUDA_CHECK(cudaMemcpyAsync(so.p, h.seq_of.p, h.n_tokens * 4, cudaMemcpyDeviceToDevice, s));
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
        h.tokens = std::move(t);
        h.seq_of = std::move(so);
        h.tok_cap = cap;
        changed = true;
    }
    if (need_seq > h.seq_cap) {
        int cap = std::max(need_seq, std::max(64, h.seq_cap * 2));
        DevBuf<int32_t> a(cap), b(cap);
        DevBuf<int64_t> c(cap);
        if (h.n_seqs) {
            CUDA_CHECK(cudaMemcpyAsync(a.p, h.seq_start.p, h.n_seqs * 4, cudaMemcpyDeviceToDevice, s));
            CUDA_CHECK(cudaMemcpyAsync(b.p, h.seq_len.p, h.n_seqs * 4, cudaMemcpyDeviceToDevice, s));
            CUDA_CHECK(cudaMemcpyAsync(c.p, h.seq_step.p, h.n_seqs * 8, cudaMemcpyDeviceToDevice, s));
        }
        CUDA_CHECK(cudaStreamSynchronize(s));
        h.seq_start = std::move(a);
        h.seq_len = std::move(b);
        h.seq_step = std::move(c);
        h.seq_cap = cap;
        changed = true;
    }
    if (changed) {
        LayerDesc v = desc_of(h);
        set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 1);
        CUDA_LAUNCH_CHECK();
    }
}

void DeviceStore::add_stats(const int64_t delta[6], cudaStream_t s) {
    DeviceGuard g(device_);
    add_stats_kernel<<<1, 32, 0, s>>>(desc_dev_, delta[0], delta[1], delta[2], delta[3], delta[4], delta[5]);
    CUDA_LAUNCH_CHECK();
}

void DeviceStore::set_rejected_enabled(bool on, cudaStream_t s) {
    DeviceGuard g(device_);
    rejected_enabled_ = on;
    set_store_kernel<<<1, 1, 0, s>>>(desc_dev_, max_order_, on ? 1 : 0);
    CUDA_LAUNCH_CHECK();
}

void DeviceStore::set_layer_order(int l, int order, cudaStream_t s) {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    if (order < 1 || order > kMaxOrder) throw_invalid("layer max_order out of range");
    DeviceGuard g(device_);
    HostLayer& h = layers_[l];
    h.max_order = order;
    if (order > h.idx_order) h.idx_tokens = 0;  // orders above the index's: scan the whole layer
    LayerDesc v = desc_of(h);
    set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 1);
    CUDA_LAUNCH_CHECK();
}

void DeviceStore::insert(int l, const int32_t* tokens, int n, long step, cudaStream_t s) {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    if (n <= 0) throw_invalid("insert: empty token sequence");  // datastore.cpp:10
    HostLayer& h = layers_[l];
    if (static_cast<long>(h.n_tokens) + n >= (1L << 24) || h.n_seqs + 1 >= (1 << 24))
        throw_runtime("datastore layer exceeds 2^24 tokens/sequences");
    DeviceGuard g(device_);
    grow(l, h.n_tokens + n, h.n_seqs + 1, s);
    if (staging_at_ + n > staging_[staging_cur_].buf.n) {
        // ring full: continue in the other ring once its own earlier payloads have been consumed
        Staging& nx = staging_[staging_cur_ ^ 1];
        nx.drain();
        size_t cap = std::max(nx.buf.n, staging_[staging_cur_].buf.n);
        while (cap < static_cast<size_t>(n)) cap *= 2;
        if (cap > nx.buf.n) nx.buf.alloc(cap);  // nothing of nx is in flight any more
        staging_cur_ ^= 1;
        staging_at_ = 0;
    }
    Staging& rg = staging_[staging_cur_];
    std::memcpy(rg.buf.p + staging_at_, tokens, static_cast<size_t>(n) * 4);
    append_kernel<<<1, 256, 0, s>>>(desc_dev_, l, rg.buf.dev() + staging_at_, n, step);
    CUDA_LAUNCH_CHECK();
    rg.mark(s);
    staging_at_ += static_cast<size_t>(n);
    h.n_tokens += n;
    h.n_seqs += 1;
    h.lens.push_back(n);
}

void DeviceStore::clear_layer(int l, cudaStream_t s) {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    DeviceGuard g(device_);
    HostLayer& h = layers_[l];
    h.n_tokens = h.n_seqs = 0;
    h.idx_tokens = 0;  // the index buffers are kept for reuse
    h.lens.clear();
    LayerDesc v = desc_of(h);
    set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 0);
    CUDA_LAUNCH_CHECK();
}

// a deep copy (the reference's HierarchicalDatastore is copied by value: test_pipeline.cpp:170-187)
std::unique_ptr<DeviceStore> DeviceStore::clone_to(int device) const {
    {
        DeviceGuard g0(device_);
        CUDA_CHECK(cudaDeviceSynchronize());  // every enqueued append of this store has landed
    }
    auto c = std::make_unique<DeviceStore>(max_order_, depth_, device);
    DeviceGuard g(device);
    c->step_ = step_;
    c->rejected_enabled_ = rejected_enabled_;
    for (int l = 0; l < 3; ++l) {
        const HostLayer& h = layers_[l];
        HostLayer& d = c->layers_[l];
        d.max_order = h.max_order;
        c->grow(l, std::max(h.n_tokens, 1), std::max(h.n_seqs, 1), 0);
        if (h.n_tokens) {
            CUDA_CHECK(cudaMemcpy(d.tokens.p, h.tokens.p, h.n_tokens * 4, cudaMemcpyDeviceToDevice));
            CUDA_CHECK(cudaMemcpy(d.seq_of.p, h.seq_of.p, h.n_tokens * 4, cudaMemcpyDeviceToDevice));
        }
        if (h.n_seqs) {
            CUDA_CHECK(cudaMemcpy(d.seq_start.p, h.seq_start.p, h.n_seqs * 4, cudaMemcpyDeviceToDevice));
            CUDA_CHECK(cudaMemcpy(d.seq_len.p, h.seq_len.p, h.n_seqs * 4, cudaMemcpyDeviceToDevice));
            CUDA_CHECK(cudaMemcpy(d.seq_step.p, h.seq_step.p, h.n_seqs * 8, cudaMemcpyDeviceToDevice));
        }
        d.n_tokens = h.n_tokens;
        d.n_seqs = h.n_seqs;
        d.lens = h.lens;
        LayerDesc v = desc_of(d);
        set_layer_kernel<<<1, 1>>>(c->desc_dev_, l, v, 0);
        CUDA_LAUNCH_CHECK();
    }
    for (int l = 0; l < 3; ++l)
        if (layers_[l].idx_tokens > 0) c->build_index(l, 0);  // covers at least what the source's index does
    set_store_kernel<<<1, 1>>>(c->desc_dev_, max_order_, rejected_enabled_ ? 1 : 0);
    CUDA_LAUNCH_CHECK();
    {  // stats: through the host (the source may be on another GPU)
        StoreDesc hs;
        {
            DeviceGuard g0(device_);
            CUDA_CHECK(cudaMemcpy(&hs, desc_dev_, sizeof hs, cudaMemcpyDeviceToHost));
        }
        CUDA_CHECK(cudaMemcpy(c->desc_dev_->stats, hs.stats, sizeof hs.stats, cudaMemcpyHostToDevice));
    }
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaDeviceSynchronize());
    return c;
}

// layer l := n_seqs sequences (off[n_seqs + 1] into toks) with steps 0..n_seqs-1 and order max_order, in
// one upload: tokens and the per-sequence records are copied once, seq_of is filled on the device
void DeviceStore::load_layer(int l, int max_order, const int64_t* off, const int32_t* toks, int n_seqs, cudaStream_t s) {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    if (max_order < 1 || max_order > kMaxOrder) throw_invalid("layer max_order out of range");
    if (n_seqs < 0) throw_invalid("negative sequence count");
    const int64_t nt = n_seqs > 0 ? off[n_seqs] : 0;
    if (n_seqs > 0 && off[0] != 0) throw_invalid("sequence offsets must start at 0");
    for (int q = 0; q < n_seqs; ++q)
        if (off[q + 1] <= off[q]) throw_invalid("insert: empty token sequence");  // datastore.cpp:10
    if (nt >= (1L << 24) || n_seqs >= (1 << 24)) throw_runtime("datastore layer exceeds 2^24 tokens/sequences");
    DeviceGuard g(device_);
    clear_layer(l, s);
    HostLayer& h = layers_[l];
    h.max_order = max_order;
    grow(l, static_cast<int>(std::max<int64_t>(nt, 1)), std::max(n_seqs, 1), s);
    std::vector<int32_t> start(n_seqs), len(n_seqs);
    std::vector<int64_t> step(n_seqs);
    h.lens.resize(n_seqs);
    for (int q = 0; q < n_seqs; ++q) {
        start[q] = static_cast<int32_t>(off[q]);
        len[q] = h.lens[q] = static_cast<int32_t>(off[q + 1] - off[q]);
        step[q] = q;
    }
    if (n_seqs > 0) {
        CUDA_CHECK(cudaMemcpyAsync(h.tokens.p, toks, nt * 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(h.seq_start.p, start.data(), n_seqs * 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(h.seq_len.p, len.data(), n_seqs * 4, cudaMemcpyHostToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(h.seq_step.p, step.data(), n_seqs * 8, cudaMemcpyHostToDevice, s));
        fill_seq_of_kernel<<<std::min(n_seqs, 1184), 256, 0, s>>>(h.seq_of.p, h.seq_start.p, h.seq_len.p, n_seqs);
        CUDA_LAUNCH_CHECK();
    }
    h.n_tokens = static_cast<int32_t>(nt);
    h.n_seqs = n_seqs;
    LayerDesc v = desc_of(h);
    set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 0);
    CUDA_LAUNCH_CHECK();
    // the index pays off past a few thousand tokens (a scan of a small prior is as fast as a probe, and
    // building costs a sort and a host sync); DBL_STORE_INDEX_MIN overrides the threshold
    static const int64_t index_min = [] {
        const char* e = std::getenv("DBL_STORE_INDEX_MIN");
        return e ? std::atoll(e) : 4096LL;
    }();
    if (nt >= index_min) build_index(l, s);  // synchronises s
    else CUDA_CHECK(cudaStreamSynchronize(s));  // the host vectors above are pageable sources
}

void DeviceStore::lookup_lane(int32_t* buf, LaneState* lane, int d, cudaStream_t s) const {
    lookup_lane_kernel<<<1, kLookupThreads, 0, s>>>(desc_dev_, buf, lane, d);
    CUDA_LAUNCH_CHECK();
}

void DeviceStore::lookup_batch(int n_q, const int64_t* offsets, const int32_t* toks,
                               const int32_t* depths, int d_cap, int32_t* out_cands, int32_t* out_n,
                               int32_t* out_src, int32_t* out_order, cudaStream_t s) {
    if (n_q <= 0) return;
    DeviceGuard g(device_);
    for (int q = 0; q < n_q; ++q) {
        if (offsets[q + 1] <= offsets[q]) throw_invalid("lookup: empty context");  // datastore.cpp:84
        if (depths[q] > 65535) throw_invalid("lookup depth must be <= 65535");
        if (std::max(depths[q], 0) > d_cap) throw_invalid("d_cap smaller than a query depth");
    }
    const int64_t ntok = offsets[n_q];
    DevBuf<int64_t> doff(n_q + 1);
    DevBuf<int32_t> dtok(std::max<int64_t>(ntok, 1)), ddep(n_q), dc(static_cast<size_t>(n_q) * std::max(d_cap, 1)),
        dn(n_q), dsrc(n_q), dord(n_q);
    CUDA_CHECK(cudaMemcpyAsync(doff.p, offsets, (n_q + 1) * 8, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(dtok.p, toks, ntok * 4, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpyAsync(ddep.p, depths, n_q * 4, cudaMemcpyHostToDevice, s));
    lookup_batch_kernel<<<n_q, kLookupThreads, 0, s>>>(desc_dev_, doff.p, dtok.p, ddep.p, d_cap, dc.p,
                                                       dn.p, dsrc.p, dord.p);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaMemcpyAsync(out_cands, dc.p, dc.bytes(), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(out_n, dn.p, n_q * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(out_src, dsrc.p, n_q * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(out_order, dord.p, n_q * 4, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
}

double DeviceStore::profile_lookup(const int32_t* ctx, int L, int d, int iters) {
    DeviceGuard g(device_);
    if (d > 65535) throw_invalid("lookup depth must be <= 65535");
    const int dcap = std::max(d, 1);
    DevBuf<int64_t> doff(2);
    DevBuf<int32_t> dtok(L), ddep(1), dc(dcap), dn(1), dsrc(1), dord(1);
    const int64_t off[2] = {0, L};
    CUDA_CHECK(cudaMemcpy(doff.p, off, 16, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(dtok.p, ctx, static_cast<size_t>(L) * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(ddep.p, &d, 4, cudaMemcpyHostToDevice));
    cudaStream_t s;
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
    auto launch = [&] {
        lookup_batch_kernel<<<1, kLookupThreads, 0, s>>>(desc_dev_, doff.p, dtok.p, ddep.p, dcap, dc.p, dn.p, dsrc.p, dord.p);
    };
    for (int i = 0; i < 3; ++i) launch();
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaEventRecord(e0, s));
    for (int i = 0; i < iters; ++i) launch();
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaEventRecord(e1, s));
    CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    return 1e3 * static_cast<double>(ms) / iters;
}

void DeviceStore::stats(int64_t out[6], cudaStream_t s) const {
    DeviceGuard g(device_);
    StoreDesc h;
    CUDA_CHECK(cudaMemcpyAsync(&h, desc_dev_, sizeof h, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    for (int i = 0; i < 6; ++i) out[i] = static_cast<int64_t>(h.stats[i]);
}

void DeviceStore::layer_info(int l, int64_t* n_seqs, int64_t* n_tokens, int64_t* occ) const {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    const HostLayer& h = layers_[l];
    if (n_seqs) *n_seqs = h.n_seqs;
    if (n_tokens) *n_tokens = h.n_tokens;
    if (occ) {
        int64_t total = 0;
        for (int len : h.lens)
            for (int k = 1; k <= h.max_order; ++k)
                if (len >= k) total += len - k + 1;
        *occ = total;
    }
}

void DeviceStore::layer_read(int l, int32_t* toks, int64_t tok_cap, int32_t* lens, int64_t* steps,
                             int64_t seq_cap, cudaStream_t s) const {
    if (l < 0 || l > 2) throw_invalid("bad datastore layer");
    const HostLayer& h = layers_[l];
    if (tok_cap < h.n_tokens || seq_cap < h.n_seqs) throw_invalid("layer_read: buffers too small");
    DeviceGuard g(device_);
    if (h.n_tokens) CUDA_CHECK(cudaMemcpyAsync(toks, h.tokens.p, h.n_tokens * 4, cudaMemcpyDeviceToHost, s));
    if (h.n_seqs) {
        CUDA_CHECK(cudaMemcpyAsync(lens, h.seq_len.p, h.n_seqs * 4, cudaMemcpyDeviceToHost, s));
        CUDA_CHECK(cudaMemcpyAsync(steps, h.seq_step.p, h.n_seqs * 8, cudaMemcpyDeviceToHost, s));
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace dbl
