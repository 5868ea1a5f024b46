// Retrieval kernels (K1 lookup, K1b insert) and the DeviceStore host object.
// Semantics: HierarchicalDatastore::lookup / NGramIndex::insert (datastore.cpp:9-132).
#include <algorithm>
#include <cstring>

#include "store.cuh"

namespace dbl {

namespace {

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
    __shared__ Key s_red[kWarps];
    __shared__ Key s_best[3][kMaxOrder + 1];
    __shared__ int s_pld[kWarps];
    __shared__ int s_pld_end[kMaxOrder + 1];
    __shared__ int s_choice[4];  // src, order, from, layer-seq
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = sd->max_order;
    const int nkey = min(N, L);
    if (tid < kMaxOrder) s_key[tid] = tid < nkey ? ctx[L - 1 - tid] : -1;
    __syncthreads();

    // ---- layer scans: for each layer, the best occurrence per order n (all orders in one pass)
    for (int l = 0; l < 3; ++l) {
        const LayerDesc ly = sd->layer[l];
        const bool enabled = (l != 2 || sd->rejected_enabled) && ly.n_tokens > 0;
        const int Nl = min(nkey, ly.max_order);
        Key best[kMaxOrder + 1];
#pragma unroll
        for (int n = 0; n <= kMaxOrder; ++n) best[n] = Key{0ull, 0ull};
        if (enabled && Nl >= 1) {
            const int k0 = s_key[0];
            for (int p = tid; p < ly.n_tokens; p += kLookupThreads) {
                if (__ldg(ly.tokens + p) != k0) continue;  // cheap filter: last token must match
                const int q = __ldg(ly.seq_of + p);
                const int st = __ldg(ly.seq_start + q);
                const int len = __ldg(ly.seq_len + q);
                const int e = p - st;
                const int remaining = len - e - 1;
                const int avail = min(remaining, d);
                if (avail <= 0) continue;
                int m = 1;
                const int mmax = min(Nl, e + 1);
                while (m < mmax && __ldg(ly.tokens + p - m) == s_key[m]) ++m;
                Key k;
                k.hi = static_cast<unsigned long long>(__ldg(ly.seq_step + q)) ^ 0x8000000000000000ull;
                k.lo = (static_cast<unsigned long long>(avail) << 48) |
                       (static_cast<unsigned long long>(q) << 24) | static_cast<unsigned long long>(e);
#pragma unroll
                for (int n = 1; n <= kMaxOrder; ++n)
                    if (n <= m && key_gt(k, best[n])) best[n] = k;
            }
        }
        for (int n = 1; n <= kMaxOrder; ++n) {  // block max-reduce per order (uniform loop)
            if (n > N) break;
            Key k = key_shfl_max(best[n]);
            if (lane == 0) s_red[warp] = k;
            __syncthreads();
            if (warp == 0) {
                Key r = lane < kWarps ? s_red[lane] : Key{0ull, 0ull};
                r = key_shfl_max(r);
                if (lane == 0) s_best[l][n] = r;
            }
            __syncthreads();
        }
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
__global__ void set_stats_kernel(StoreDesc* sd, const StoreDesc* src) {
    if (threadIdx.x < 6) sd->stats[threadIdx.x] = src->stats[threadIdx.x];
}
__global__ void set_store_kernel(StoreDesc* sd, int max_order, int rej) {
    sd->max_order = max_order;
    sd->rejected_enabled = rej;
}

}  // namespace

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
        LayerDesc v{h.tokens.p, h.seq_of.p, h.seq_start.p, h.seq_len.p, h.seq_step.p,
                    h.n_tokens, h.n_seqs, h.max_order, 0};
        set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 1);
        CUDA_LAUNCH_CHECK();
    }
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
    LayerDesc v{h.tokens.p, h.seq_of.p, h.seq_start.p, h.seq_len.p, h.seq_step.p,
                h.n_tokens, h.n_seqs, h.max_order, 0};
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
    h.lens.clear();
    LayerDesc v{h.tokens.p, h.seq_of.p, h.seq_start.p, h.seq_len.p, h.seq_step.p, 0, 0, h.max_order, 0};
    set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 0);
    CUDA_LAUNCH_CHECK();
}

// a deep copy (the reference's HierarchicalDatastore is copied by value: test_pipeline.cpp:170-187)
std::unique_ptr<DeviceStore> DeviceStore::clone() const {
    auto c = std::make_unique<DeviceStore>(max_order_, depth_, device_);
    DeviceGuard g(device_);
    CUDA_CHECK(cudaDeviceSynchronize());  // every enqueued append of this store has landed
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
        LayerDesc v{d.tokens.p, d.seq_of.p, d.seq_start.p, d.seq_len.p, d.seq_step.p, d.n_tokens, d.n_seqs,
                    d.max_order, 0};
        set_layer_kernel<<<1, 1>>>(c->desc_dev_, l, v, 0);
        CUDA_LAUNCH_CHECK();
    }
    set_store_kernel<<<1, 1>>>(c->desc_dev_, max_order_, rejected_enabled_ ? 1 : 0);
    CUDA_LAUNCH_CHECK();
    set_stats_kernel<<<1, 32>>>(c->desc_dev_, desc_dev_);
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
    LayerDesc v{h.tokens.p, h.seq_of.p, h.seq_start.p, h.seq_len.p, h.seq_step.p, h.n_tokens, h.n_seqs, h.max_order, 0};
    set_layer_kernel<<<1, 1, 0, s>>>(desc_dev_, l, v, 0);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaStreamSynchronize(s));  // the host vectors above are pageable sources
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
