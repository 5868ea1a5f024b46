// K3' — the sampled (temperature > 0) decode path on the device.
//
// The reference's stochastic loop (speculation.cpp:7-52 accept_with_model, pipeline.cpp:91-140
// finish_round, harness.cpp:233-330 AR / serial SD) consumes full ProbVector rows and mt19937_64
// streams.  Here each acceptance step is ONE block (kNT threads) over fp64 rows resident in HBM:
//   * elementwise work (tempered's pow / normalise, residual max(0, p - q)) is spread over the block
//     — identical per element to the reference's loop;
//   * sums and the inverse-CDF scan follow the reference's sequential order on one thread when the
//     vocabulary is small (<= kExactVocab, e.g. the table models of config 1) or exact sampling is on
//     (dbl_set_exact_sampling), so every decision and token is bit-identical to the reference; by
//     default wide vocabularies use coalesced fixed-order reductions, a two-level warp-segment scan
//     and fp32 tempering (pow via exp2/log2) — deterministic, same law, ~1.2 MB rows at block bandwidth;
//   * every uniform() is drawn by thread 0 from the lane's mt19937_64 state, staged in shared memory
//     for the kernel's lifetime, in exactly the reference's draw order.
#include "rng.cuh"
#include "sampling.cuh"

namespace dbl {

namespace {

constexpr int kNT = 1024;
constexpr int kExactVocab = 4096;
// reference-exact sampling at every vocabulary size (dbl_set_exact_sampling): the sequential sums,
// scan and fp64 pow of the small-vocabulary path for wide rows too — bit-identical decisions with the
// reference at e.g. V = 151,936, at ~0.5 ms of single-thread fp64 work per row
__device__ int g_exact_sampling = 0;
__device__ __forceinline__ bool exact_path(int n) { return n <= kExactVocab || g_exact_sampling != 0; }

struct Blk {
    double red[kNT];
    int last[kNT];
    double f, u;
    int i0, i1;
};

__device__ __forceinline__ double blk_bcast(Blk& sh, double v, bool from0) {
    if (from0 && threadIdx.x == 0) sh.u = v;
    __syncthreads();
    const double r = sh.u;
    __syncthreads();
    return r;
}

// sum of w[0, n) in the reference's order (n <= kExactVocab) or a fixed chunked tree
__device__ double blk_sum(Blk& sh, const double* w, int n) {
    const int t = threadIdx.x;
    if (exact_path(n)) {
        if (t == 0) {
            double a = 0.0;
            for (int i = 0; i < n; ++i) a += w[i];
            sh.f = a;
        }
    } else {  // thread t sums the elements t, t + kNT, ... (coalesced), then a fixed tree
        double a = 0.0;
        for (int i = t; i < n; i += kNT) a += w[i];
        sh.red[t] = a;
        __syncthreads();
        for (int s = kNT / 2; s > 0; s >>= 1) {
            if (t < s) sh.red[t] += sh.red[t + s];
            __syncthreads();
        }
        if (t == 0) sh.f = sh.red[0];
    }
    __syncthreads();
    const double r = sh.f;
    __syncthreads();
    return r;
}

// the inverse-CDF scan of sample / sample_from (model.cpp:83-97, verification.cpp:25-38): the first
// positive entry whose running sum exceeds u, else the last positive entry (rounding slack), else -1
__device__ int blk_pick(Blk& sh, const double* w, int n, double u) {
    const int t = threadIdx.x;
    if (exact_path(n)) {
        if (t == 0) {
            double acc = 0.0;
            int last = -1, r = -2;
            for (int i = 0; i < n; ++i) {
                if (w[i] <= 0.0) continue;
                last = i;
                acc += w[i];
                if (u < acc) { r = i; break; }
            }
            sh.i0 = r == -2 ? last : r;
        }
    } else {
        // warp v owns the contiguous segment [v*seg, (v+1)*seg); its lanes read it 32 elements at a time
        constexpr int kW = kNT / 32;
        const int v = t >> 5, ln = t & 31;
        const int seg = ((n + kW - 1) / kW + 31) & ~31;
        const int lo = v * seg, hi = min(n, lo + seg);
        double a = 0.0;
        int last = -1;
        for (int i = lo + ln; i < hi; i += 32)
            if (w[i] > 0.0) {
                a += w[i];
                last = i;
            }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, off);
            last = max(last, __shfl_xor_sync(0xffffffffu, last, off));
        }
        if (ln == 0) {
            sh.red[v] = a;
            sh.last[v] = last;
        }
        __syncthreads();
        if (t == 0) {
            double acc = 0.0;
            int sel = -1, glast = -1;
            for (int k = 0; k < kW; ++k) {
                if (sh.last[k] < 0) continue;
                glast = sh.last[k];
                if (u < acc + sh.red[k]) { sel = k; break; }
                acc += sh.red[k];
            }
            sh.i1 = sel;
            sh.f = acc;
            sh.i0 = glast;
        }
        __syncthreads();
        if (sh.i1 == v) {  // the selected warp scans its segment: inclusive warp prefix per 32-element block
            double base = sh.f;
            int r = sh.last[v];
            for (int i0 = lo; i0 < hi; i0 += 32) {
                const int i = i0 + ln;
                const double x = i < hi ? w[i] : 0.0;
                const double val = x > 0.0 ? x : 0.0;
                double pre = val;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const double o = __shfl_up_sync(0xffffffffu, pre, off);
                    if (ln >= off) pre += o;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, val > 0.0 && u < base + pre);
                if (hit) {
                    r = i0 + __ffs(hit) - 1;
                    break;
                }
                base += __shfl_sync(0xffffffffu, pre, 31);
            }
            if (ln == 0) sh.i0 = r;
        }
    }
    __syncthreads();
    const int r = sh.i0;
    __syncthreads();
    return r;
}

// out = tempered(dist, T) (model.cpp:55-68); false when the tempered mass is not positive
__device__ bool blk_tempered(Blk& sh, const double* dist, double* out, int n, double T) {
    if (T == 1.0) {  // the reference returns dist itself
        for (int i = threadIdx.x; i < n; i += kNT) out[i] = dist[i];
        __syncthreads();
        return true;
    }
    const double inv = 1.0 / T;
    if (exact_path(n)) {
        for (int i = threadIdx.x; i < n; i += kNT) out[i] = dist[i] > 0.0 ? pow(dist[i], inv) : 0.0;
    } else {  // fp32 pow (exp2 . log2): rows of 1e5+ entries at block rate; no reference to match here
        const float invf = static_cast<float>(inv);
        for (int i = threadIdx.x; i < n; i += kNT) {
            const double x = dist[i];
            out[i] = x > 0.0 ? static_cast<double>(exp2f(log2f(static_cast<float>(x)) * invf)) : 0.0;
        }
    }
    __syncthreads();
    const double sum = blk_sum(sh, out, n);
    if (sum <= 0.0) return false;
    for (int i = threadIdx.x; i < n; i += kNT) out[i] /= sum;
    __syncthreads();
    return true;
}

__device__ __forceinline__ double blk_uniform(Blk& sh, DevRng& g) {
    return blk_bcast(sh, threadIdx.x == 0 ? mt_uniform(g) : 0.0, true);
}

// residual_sample_point_mass (verification.cpp:52-58): p with p[x] removed, via scratch w.
// Returns the token, or -1 with *err set.
__device__ int blk_residual_point(Blk& sh, const double* p, int n, int x, double* w, DevRng& g, int* err) {
    for (int i = threadIdx.x; i < n; i += kNT) w[i] = i == x ? 0.0 : p[i];
    __syncthreads();
    const double total = blk_sum(sh, w, n);
    if (total <= 0.0) { *err = kSampResidualZero; return -1; }
    const double u = blk_uniform(sh, g) * total;
    return blk_pick(sh, w, n, u);
}

// residual_sample (verification.cpp:40-50): max(0, p - q)
__device__ int blk_residual(Blk& sh, const double* p, const double* q, int n, double* w, DevRng& g, int* err) {
    for (int i = threadIdx.x; i < n; i += kNT) w[i] = fmax(0.0, p[i] - q[i]);
    __syncthreads();
    const double total = blk_sum(sh, w, n);
    if (total <= 0.0) { *err = kSampResidualZero; return -1; }
    const double u = blk_uniform(sh, g) * total;
    return blk_pick(sh, w, n, u);
}

// sample (model.cpp:83-97) at T > 0: eff = tempered(dist) into `eff`, one draw, scan
__device__ int blk_sample(Blk& sh, const double* dist, double* eff, int n, double T, DevRng& g, int* err) {
    if (!blk_tempered(sh, dist, eff, n, T)) { *err = kSampDegenerate; return -1; }
    const double u = blk_uniform(sh, g);
    const int tok = blk_pick(sh, eff, n, u);
    if (tok < 0) *err = kSampDegenerate;
    return tok;
}

// accept_with_model at T > 0 over rows D(0..c) and candidates cand[0..c) (speculation.cpp:14-51).
// Row i's eff is written to E(i) (E may alias one scratch row when the rows are not kept).
// Returns matched s; *tok = the continuation token.
template <class DRow, class ERow>
__device__ int blk_accept(Blk& sh, DRow D, ERow E, const int32_t* cand, int c, int vocab, double T, DevRng& g,
                          double* w, int* tok, int* err) {
    int s = 0;
    bool rejected = false;
    while (s < c) {
        const int x = cand[s];
        // speculation.cpp:19 breaks here and then indexes a point-mass residual at x: undefined in
        // the reference for T > 0, an argument error here
        if (x < 0 || x >= vocab) { *err = kSampInvalid; return s; }
        if (!blk_tempered(sh, D(s), E(s), vocab, T)) { *err = kSampDegenerate; return s; }
        const double u = blk_uniform(sh, g);
        if (!(u < E(s)[x])) { rejected = true; break; }
        ++s;
    }
    if (rejected) *tok = blk_residual_point(sh, E(s), vocab, cand[s], w, g, err);
    else *tok = blk_sample(sh, D(s), E(s), vocab, T, g, err);
    return s;
}

__device__ __forceinline__ void rng_load(DevRng& dst, const DevRng* src) {
    for (int i = threadIdx.x; i < 312; i += kNT) dst.mt[i] = src->mt[i];
    if (threadIdx.x == 0) dst.idx = src->idx;
}
__device__ __forceinline__ void rng_store(DevRng* dst, const DevRng& src) {
    __syncthreads();
    for (int i = threadIdx.x; i < 312; i += kNT) dst->mt[i] = src.mt[i];
    if (threadIdx.x == 0) dst->idx = src.idx;
}

__global__ void seed_rng_kernel(DevRng* g, uint64_t seed) { mt_seed(*g, seed); }
__global__ void derive_rngs_kernel(DevRng* g, uint64_t seed, uint64_t round) {
    const int lane = threadIdx.x;
    if (lane < 3) mt_seed(g[lane], derived_seed(seed, round, static_cast<uint64_t>(lane)));
}

__global__ void __launch_bounds__(kNT) draft_accept_sampled_kernel(
    const double* __restrict__ dist, int32_t* buf, LaneState* lane, int vocab, RoundResult* rr, int seg, int L0,
    double* chain, int chain_cap, DevRng* rng_g, double T, double* scratch) {
    __shared__ Blk sh;
    __shared__ DevRng g;
    rng_load(g, rng_g);
    const int L = lane->L, c = lane->c, row0 = lane->row0;
    const int base = L - L0;
    const size_t V = static_cast<size_t>(vocab);
    __syncthreads();
    int err = 0, tok = -1, s = 0;
    if (base + c + 1 > chain_cap) {
        err = kSampCapacity;
    } else {
        auto D = [&](int i) { return dist + static_cast<size_t>(L - 1 + i - row0) * V; };
        auto E = [&](int i) { return chain + static_cast<size_t>(base + i) * V; };
        s = blk_accept(sh, D, E, buf + L, c, vocab, T, g, scratch, &tok, &err);
    }
    rng_store(rng_g, g);
    if (threadIdx.x != 0) return;
    if (err) {
        lane->error = err;
        rr->draft_error = err;
        tok = 0;
    }
    buf[L + s] = tok;
    if (base + s + 1 <= kMaxRoundTokens)
        for (int i = 0; i <= s; ++i) rr->draft_tokens[base + i] = buf[L + i];
    else
        rr->draft_error = kSampCapacity;
    rr->segs[seg] = SegRecord{s, s + 1, lane->src, lane->order};
    rr->n_segs = seg + 1;
    const int Ln = L + s + 1;
    rr->draft_L = Ln;
    lane->L = Ln;
    lane->c = 0;
    lane->kv_len = Ln - 1;
    lane->row0 = Ln - 1;
    lane->src = DBL_SRC_MISS;
    lane->order = 0;
}

__global__ void __launch_bounds__(kNT) target_accept_sampled_kernel(
    const double* __restrict__ dist, const int32_t* __restrict__ buf, LaneState* lane, int vocab, int nc,
    RoundResult* rr, const double* __restrict__ spec_probs, DevRng* rng_t, DevRng* rng_v, double T, int serial,
    double* scratch) {
    __shared__ Blk sh;
    __shared__ DevRng gt, gv;
    rng_load(gt, rng_t);
    rng_load(gv, rng_v);
    const int L = lane->L, c = lane->c, row0 = lane->row0;
    const int n_spec = L - nc;
    const size_t V = static_cast<size_t>(vocab);
    double* ver = scratch;
    double* w = scratch + V;
    double* eff = scratch + 2 * V;
    auto D = [&](int i) { return dist + static_cast<size_t>(nc - 1 + i - row0) * V; };
    __syncthreads();
    // finish_round: verify_against_target over tempered target rows (pipeline.cpp:110-119,
    // verification.cpp:60-78) and the residual correction on a reject (:136-139)
    int err = 0, rej = -1, corr = -1;
    for (int k = 0; k < n_spec && !err; ++k) {
        if (!blk_tempered(sh, D(k), ver, vocab, T)) { err = kSampDegenerate; break; }
        const int x = buf[nc + k];
        if (x < 0 || x >= vocab) { err = kSampInvalid; break; }
        const double qx = spec_probs[static_cast<size_t>(k) * V + x];
        if (qx <= 0.0) { err = kSampInvalid; break; }  // "draft mass zero on emitted token"
        const double a = fmin(1.0, ver[x] / qx);
        if (blk_uniform(sh, gv) >= a) { rej = k; break; }
    }
    if (!err && rej >= 0) corr = blk_residual(sh, ver, spec_probs + static_cast<size_t>(rej) * V, vocab, w, gv, &err);
    // the target's own continuation
    int s = 0, tok = -1;
    if (serial) {
        // run_serial_sd: all accepted -> sample(dists.back(), rng_v) (harness.cpp:322-326)
        if (!err && rej < 0) tok = blk_sample(sh, D(n_spec), eff, vocab, T, gv, &err);
    } else if (!err) {
        // do_target: accept_with_model(dists[n_spec:], cands, rng_t) (pipeline.cpp:64-67)
        auto Dx = [&](int i) { return D(n_spec + i); };
        auto Ex = [&](int) { return eff; };
        s = blk_accept(sh, Dx, Ex, buf + L, c, vocab, T, gt, w, &tok, &err);
    }
    rng_store(rng_t, gt);
    rng_store(rng_v, gv);
    if (threadIdx.x != 0) return;
    if (c + 1 > kMaxRoundTokens) {  // host-validated; never write past the round record
        lane->error = kSampCapacity;
        rr->target_error = kSampCapacity;
        rr->ext_c = 0;
        return;
    }
    rr->tgt_rej = rej;
    rr->tgt_correction = corr;
    for (int i = 0; i < s; ++i) rr->ext_emitted[i] = buf[L + i];
    rr->ext_emitted[s] = tok;
    for (int i = 0; i < c; ++i) rr->ext_cands[i] = buf[L + i];
    rr->ext_matched = s;
    rr->ext_source = lane->src;
    rr->ext_order = lane->order;
    rr->ext_c = c;
    if (err) {
        lane->error = err;
        rr->target_error = err;
    }
    lane->kv_len = L + c;
}

__global__ void __launch_bounds__(kNT) ar_sample_kernel(const double* __restrict__ dist, int32_t* buf,
                                                        LaneState* lane, int vocab, DevRng* rng_g, double T,
                                                        double* scratch, int32_t* out_host, int i) {
    __shared__ Blk sh;
    __shared__ DevRng g;
    rng_load(g, rng_g);
    const int L = lane->L, row0 = lane->row0;
    __syncthreads();
    int err = 0;
    const int tok = blk_sample(sh, dist + static_cast<size_t>(L - 1 - row0) * vocab, scratch, vocab, T, g, &err);
    rng_store(rng_g, g);
    if (threadIdx.x != 0) return;
    buf[L] = err ? 0 : tok;
    out_host[i] = err ? -err - 1 : tok;
    if (err) lane->error = err;
    lane->L = L + 1;
    lane->c = 0;
    lane->kv_len = L;
    lane->row0 = L;
}

// logits rows (relative to the forward's first processed position) -> fp64 softmax rows of
// positions [row0, L+c): p = exp(l - max) / sum, fixed-order block reductions
__global__ void __launch_bounds__(kNT) softmax_rows_kernel(const float* __restrict__ logits, const LaneState* lane,
                                                           int vocab, double* __restrict__ out, const int* row_base) {
    __shared__ double red[kNT];
    const int r = blockIdx.x;
    const int rows = lane->L + lane->c - lane->row0;
    if (r >= rows) return;
    const int lrow = row_base ? *row_base + lane->row0 + r : lane->row0 - lane->start + r;
    const float* l = logits + static_cast<size_t>(lrow) * vocab;
    double* o = out + static_cast<size_t>(r) * vocab;
    const int t = threadIdx.x;
    double m = -INFINITY;
    for (int i = t; i < vocab; i += kNT) m = fmax(m, static_cast<double>(l[i]));
    red[t] = m;
    __syncthreads();
    for (int s = kNT / 2; s > 0; s >>= 1) {
        if (t < s) red[t] = fmax(red[t], red[t + s]);
        __syncthreads();
    }
    m = red[0];
    __syncthreads();
    double a = 0.0;
    const float mf = static_cast<float>(m);
    for (int i = t; i < vocab; i += kNT) {
        const double e = static_cast<double>(__expf(l[i] - mf));
        o[i] = e;
        a += e;
    }
    red[t] = a;
    __syncthreads();
    for (int s = kNT / 2; s > 0; s >>= 1) {
        if (t < s) red[t] += red[t + s];
        __syncthreads();
    }
    const double inv = 1.0 / red[0];
    for (int i = t; i < vocab; i += kNT) o[i] *= inv;
}

}  // namespace

void raise_sample_error(int code) {
    switch (code) {
        case kSampCapacity: throw_runtime("draft chain exceeds the round record");
        case kSampInvalid: throw_invalid("draft mass zero on emitted token");      // verification.cpp:21
        case kSampResidualZero: throw_runtime("residual distribution is zero");    // verification.cpp:47,56
        default: throw_runtime("degenerate distribution");                         // model.cpp:65,96
    }
}

void Model::dists(Lane& lane, int max_tokens, int max_rows, double* out_dev, cudaStream_t s) {
    const size_t need = static_cast<size_t>(std::max(max_tokens, 1)) * static_cast<size_t>(vocab());
    if (lane.logit_scratch.n < need) lane.logit_scratch.alloc(need);
    logits(lane, max_tokens, lane.logit_scratch.p, s);
    launch_softmax_rows(lane.logit_scratch.p, lane.state, vocab(), out_dev, max_rows, nullptr, s);
}

void Model::dists_lanes(const std::vector<Lane*>& lanes, int max_tokens, const std::vector<int>& max_rows,
                        const std::vector<double*>& outs, cudaStream_t s) {
    for (size_t b = 0; b < lanes.size(); ++b) dists(*lanes[b], max_tokens, max_rows[b], outs[b], s);
}

void launch_softmax_rows(const float* logits, const LaneState* lane, int vocab, double* out, int max_rows,
                         const int* row_base, cudaStream_t s) {
    softmax_rows_kernel<<<std::max(max_rows, 1), kNT, 0, s>>>(logits, lane, vocab, out, row_base);
    CUDA_LAUNCH_CHECK();
}

void launch_seed_rng(DevRng* g, uint64_t seed, cudaStream_t s) {
    seed_rng_kernel<<<1, 1, 0, s>>>(g, seed);
    CUDA_LAUNCH_CHECK();
}

void launch_derive_rngs(DevRng* g, uint64_t seed, uint64_t round, cudaStream_t s) {
    derive_rngs_kernel<<<1, 32, 0, s>>>(g, seed, round);
    CUDA_LAUNCH_CHECK();
}

void launch_draft_accept_sampled(Lane& lane, RoundResult* rr, int seg, int L0, const double* dist, double* chain,
                                 int chain_cap, DevRng* rng_d, double temperature, double* scratch, cudaStream_t s) {
    draft_accept_sampled_kernel<<<1, kNT, 0, s>>>(dist, lane.buf.p, lane.state, lane.model.vocab(), rr, seg, L0,
                                                  chain, chain_cap, rng_d, temperature, scratch);
    CUDA_LAUNCH_CHECK();
}

void launch_target_accept_sampled(Lane& lane, int n_committed, RoundResult* rr, const double* dist,
                                  const double* spec_probs, DevRng* rng_t, DevRng* rng_v, double temperature,
                                  bool serial, double* scratch, cudaStream_t s) {
    target_accept_sampled_kernel<<<1, kNT, 0, s>>>(dist, lane.buf.p, lane.state, lane.model.vocab(), n_committed,
                                                   rr, spec_probs, rng_t, rng_v, temperature, serial ? 1 : 0,
                                                   scratch);
    CUDA_LAUNCH_CHECK();
}

void launch_ar_sample(Lane& lane, const double* dist, DevRng* rng, double temperature, double* scratch,
                      int32_t* out_host, int i, cudaStream_t s) {
    ar_sample_kernel<<<1, kNT, 0, s>>>(dist, lane.buf.p, lane.state, lane.model.vocab(), rng, temperature, scratch,
                                       out_host, i);
    CUDA_LAUNCH_CHECK();
}

void set_exact_sampling(bool on) {
    int n = 0, cur = 0;
    CUDA_CHECK(cudaGetDeviceCount(&n));
    CUDA_CHECK(cudaGetDevice(&cur));
    const int v = on ? 1 : 0;
    for (int d = 0; d < n; ++d) {  // every visible device's copy of the module flag
        CUDA_CHECK(cudaSetDevice(d));
        CUDA_CHECK(cudaMemcpyToSymbol(g_exact_sampling, &v, sizeof(int)));
    }
    CUDA_CHECK(cudaSetDevice(cur));
}

}  // namespace dbl
