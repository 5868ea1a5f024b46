// The verifier API (verification.hpp:30-53) and the reference's deterministic RNG
// (rng.hpp:8-35) on the device.
//
// These are API-completeness entry points over explicit probability vectors (the decode loop itself
// is greedy and never materialises distributions).  They run as single-thread fp64 kernels so every
// sum is accumulated in the reference's order and every decision — including each mt19937_64 draw —
// is bit-identical to specpar::guided_output & co.  Ragged rows (the reference's ProbVector is a
// std::vector<double> per position) are passed flattened with row offsets.
#include <cstring>
#include <memory>
#include <vector>

#include "rng.cuh"
#include "verify.cuh"

namespace dbl {

namespace {

struct Rows {  // ragged fp64 rows: row r = data[off[r], off[r+1])
    const double* data;
    const int64_t* off;
    int n;
    __device__ const double* row(int r) const { return data + off[r]; }
    __device__ int len(int r) const { return static_cast<int>(off[r + 1] - off[r]); }
};

__device__ int argmax_row(const double* p, int n, int* err) {  // model.cpp:70-81 (ties -> lowest id)
    int best = 0;
    double bp = -1.0;
    for (int i = 0; i < n; ++i)
        if (p[i] > bp) { bp = p[i]; best = i; }
    if (bp <= 0.0) *err = kErrDegenerate;
    return best;
}
// residual_sample (verification.cpp:40-50): max(0, p - q), then sample_from; q covers p's length
__device__ int residual_sample_dev(const double* p, int np, const double* q, int nq, DevRng& g, int* err) {
    if (nq < np) { *err = kErrArgument; return -1; }
    double total = 0.0;
    for (int i = 0; i < np; ++i) total += fmax(0.0, p[i] - q[i]);
    if (total <= 0.0) { *err = kErrResidualZero; return -1; }
    const double u = mt_uniform(g) * total;
    double acc = 0.0;
    int last = -1;
    for (int i = 0; i < np; ++i) {
        const double r = fmax(0.0, p[i] - q[i]);
        if (r <= 0.0) continue;
        last = i;
        acc += r;
        if (u < acc) return last;
    }
    return last;
}
// residual_sample_point_mass (verification.cpp:52-58): p with p[x] removed
__device__ int residual_point_dev(const double* p, int np, int x, DevRng& g, int* err) {
    if (x < 0 || x >= np) { *err = kErrArgument; return -1; }
    double total = 0.0;
    for (int i = 0; i < np; ++i) total += i == x ? 0.0 : p[i];
    if (total <= 0.0) { *err = kErrResidualZero; return -1; }
    const double u = mt_uniform(g) * total;
    double acc = 0.0;
    int last = -1;
    for (int i = 0; i < np; ++i) {
        const double w = i == x ? 0.0 : p[i];
        if (w <= 0.0) continue;
        last = i;
        acc += w;
        if (u < acc) return last;
    }
    return last;
}
// accept_prob (verification.cpp:19-23)
__device__ double accept_prob_dev(const double* p, int np, const double* q, int nq, int x, int* err) {
    if (x < 0 || x >= nq || x >= np) { *err = kErrArgument; return 0.0; }
    const double qx = q[x];
    if (qx <= 0.0) { *err = kErrDraftMassZero; return 0.0; }
    return fmin(1.0, p[x] / qx);
}

__global__ void rng_seed_kernel(DevRng* g, uint64_t seed) { mt_seed(*g, seed); }
__global__ void rng_uniform_kernel(DevRng* g, double* out, int n) {
    for (int i = 0; i < n; ++i) out[i] = mt_uniform(*g);
}

struct VerifyIO {  // results written by the kernels
    int err;
    int first_reject;  // -1 = none
    int accepted_len;
    int kind;
    int n_committed;
    int token;
    double value;
};

__global__ void accept_prob_kernel(Rows p, Rows q, int x, VerifyIO* io) {
    io->err = 0;
    io->value = accept_prob_dev(p.row(0), p.len(0), q.row(0), q.len(0), x, &io->err);
}
__global__ void residual_kernel(Rows p, Rows q, int x, DevRng* g, VerifyIO* io) {
    io->err = 0;
    io->token = x >= 0 ? residual_point_dev(p.row(0), p.len(0), x, *g, &io->err)
                       : residual_sample_dev(p.row(0), p.len(0), q.row(0), q.len(0), *g, &io->err);
}

// verify_against_target (verification.cpp:60-78)
__device__ void verify_dev(const int32_t* draft, int n_draft, Rows dp, Rows tp, double temperature, DevRng& g,
                           VerifyIO* io) {
    io->first_reject = -1;
    if (tp.n < n_draft) { io->err = kErrArgument; return; }
    for (int k = 0; k < n_draft; ++k) {
        if (temperature == 0.0) {
            if (draft[k] != argmax_row(tp.row(k), tp.len(k), &io->err) || io->err) {
                if (!io->err) io->first_reject = k;
                return;
            }
        } else {
            if (k >= dp.n) { io->err = kErrArgument; return; }
            const double a = accept_prob_dev(tp.row(k), tp.len(k), dp.row(k), dp.len(k), draft[k], &io->err);
            if (io->err) return;
            if (mt_uniform(g) >= a) {
                io->first_reject = k;
                return;
            }
        }
    }
}
__global__ void verify_kernel(const int32_t* draft, int n_draft, Rows dp, Rows tp, double temperature, DevRng* g,
                              VerifyIO* io) {
    io->err = 0;
    verify_dev(draft, n_draft, dp, tp, temperature, *g, io);
}

// guided_output (verification.cpp:80-132)
__global__ void guided_kernel(const int32_t* draft, int n_draft, Rows dp, const int32_t* gtok, int n_gtok, Rows gp,
                              int first_reject, double temperature, DevRng* g, int32_t* committed, int cap,
                              VerifyIO* io) {
    io->err = 0;
    int n = 0;
    auto push = [&](int32_t t) {
        if (n < cap) committed[n] = t;
        ++n;
    };
    if (first_reject < 0) {
        io->accepted_len = n_draft;
        for (int i = 0; i < n_draft; ++i) push(draft[i]);
        io->kind = kAllAccepted;
        bool covers = temperature == 0.0 && n_gtok > n_draft;
        for (int i = 0; covers && i < n_draft; ++i) covers = draft[i] == gtok[i];
        if (covers) {
            for (int i = n_draft; i < n_gtok; ++i) push(gtok[i]);
            io->kind = kExtension;
        }
        io->n_committed = n;
        return;
    }
    const int i = first_reject;
    if (i > n_draft) { io->err = kErrArgument; return; }
    io->accepted_len = i;
    for (int k = 0; k < i; ++k) push(draft[k]);
    if (temperature == 0.0) {
        if (i < n_gtok) {
            for (int k = i; k < n_gtok; ++k) push(gtok[k]);
        } else if (i < gp.n) {
            push(argmax_row(gp.row(i), gp.len(i), &io->err));
        } else {
            io->err = kErrUncovered;
            return;
        }
        io->kind = kCorrection;
        io->n_committed = n;
        return;
    }
    if (i >= gp.n) { io->err = kErrUncovered; return; }
    if (i >= dp.n) { io->err = kErrArgument; return; }
    push(residual_sample_dev(gp.row(i), gp.len(i), dp.row(i), dp.len(i), *g, &io->err));
    io->kind = kResidualCorrection;
    io->n_committed = n;
}

// tempered (model.cpp:55-68): p^(1/T) over the positive entries, renormalised in index order; T = 1
// returns the row unchanged
__device__ bool tempered_dev(const double* p, int n, double T, double* out) {
    if (T == 1.0) {
        for (int i = 0; i < n; ++i) out[i] = p[i];
        return true;
    }
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        out[i] = p[i] > 0.0 ? pow(p[i], 1.0 / T) : 0.0;
        sum += out[i];
    }
    if (sum <= 0.0) return false;
    for (int i = 0; i < n; ++i) out[i] /= sum;
    return true;
}
// sample (model.cpp:83-97) at T > 0 over the tempered row `eff` (already computed): one draw
__device__ int sample_eff_dev(const double* eff, int n, DevRng& g, int* err) {
    const double u = mt_uniform(g);
    double acc = 0.0;
    int last = -1;
    for (int i = 0; i < n; ++i) {
        if (eff[i] <= 0.0) continue;
        last = i;
        acc += eff[i];
        if (u < acc) return last;
    }
    if (last < 0) *err = kErrDegenerate;
    return last;
}

// argmax_token (model.cpp:70-81) as a block reduction: each thread keeps the strict-greater running
// max of its strided slice (so the lowest id wins ties inside the slice), then (max, lowest id) pairs
// are merged by warp shuffles and across warps.  NaN entries never compare greater, as in the scan.
constexpr int kArgThreads = 1024;
__global__ void __launch_bounds__(kArgThreads) argmax_rows_kernel(Rows p, int32_t* out, int* err) {
    __shared__ double sv[kArgThreads / 32];
    __shared__ int si[kArgThreads / 32];
    const double* row = p.row(blockIdx.x);
    const int n = p.len(blockIdx.x);
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += kArgThreads)
        if (row[i] > bv) { bv = row[i]; bi = i; }
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_down_sync(0xffffffffu, bv, o);
        const int i = __shfl_down_sync(0xffffffffu, bi, o);
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sv[w] = bv; si[w] = bi; }
    __syncthreads();
    if (w == 0) {
        bv = sv[l];
        bi = si[l];
        for (int o = 16; o; o >>= 1) {
            const double v = __shfl_down_sync(0xffffffffu, bv, o);
            const int i = __shfl_down_sync(0xffffffffu, bi, o);
            if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
        }
        if (l == 0) {
            if (!(bv > 0.0)) *err = kErrDegenerate;  // best_p <= 0 (also n == 0)
            out[blockIdx.x] = bv > 0.0 ? bi : 0;
        }
    }
}

__global__ void tempered_kernel(Rows p, double T, double* out, VerifyIO* io) {
    io->err = 0;
    if (!tempered_dev(p.row(0), p.len(0), T, out)) io->err = kErrDegenerate;
}
__global__ void sample_kernel(Rows p, double T, DevRng* g, double* eff, VerifyIO* io) {
    io->err = 0;
    if (T == 0.0) {
        io->token = argmax_row(p.row(0), p.len(0), &io->err);
        return;
    }
    if (!tempered_dev(p.row(0), p.len(0), T, eff)) { io->err = kErrDegenerate; return; }
    io->token = sample_eff_dev(eff, p.len(0), *g, &io->err);
}

// accept_with_model (speculation.cpp:7-52) over ragged rows D (|cands| + 1 of them).  eff rows (T > 0)
// are written to E at D's offsets; greedy probs are the D rows themselves (the host copies them).
// io: accepted_len = matched, n_committed = |emitted|, first_reject = |probs|.
__global__ void accept_model_kernel(Rows D, const int32_t* cand, int c, double T, DevRng* g, double* E,
                                    int32_t* emitted, VerifyIO* io) {
    io->err = 0;
    const bool greedy = T == 0.0;
    int s = 0, n_probs = 0;
    while (s < c) {
        const double* dist = D.row(s);
        const int n = D.len(s), x = cand[s];
        if (x < 0 || x >= n) break;
        if (greedy) {
            const int a = argmax_row(dist, n, &io->err);
            if (io->err) return;
            if (x != a) break;
            ++n_probs;
        } else {
            double* eff = E + D.off[s];
            if (!tempered_dev(dist, n, T, eff)) { io->err = kErrDegenerate; return; }
            const bool acc = mt_uniform(*g) < eff[x];
            ++n_probs;
            if (!acc) break;
        }
        emitted[s] = x;
        ++s;
    }
    io->accepted_len = s;
    if (s < c) {
        if (greedy) {
            emitted[s] = argmax_row(D.row(s), D.len(s), &io->err);
            ++n_probs;
        } else {
            // probs.back() is row s's eff; with an out-of-range candidate the reference reads the
            // previous row (or an empty vector) — an argument error here
            if (n_probs != s + 1 || cand[s] < 0 || cand[s] >= D.len(s)) { io->err = kErrArgument; return; }
            emitted[s] = residual_point_dev(E + D.off[s], D.len(s), cand[s], *g, &io->err);
        }
    } else {
        const double* dist = D.row(s);
        const int n = D.len(s);
        if (greedy) {
            emitted[s] = argmax_row(dist, n, &io->err);
        } else {
            double* eff = E + D.off[s];
            if (!tempered_dev(dist, n, T, eff)) { io->err = kErrDegenerate; return; }
            emitted[s] = sample_eff_dev(eff, n, *g, &io->err);
        }
        ++n_probs;
    }
    io->n_committed = s + 1;
    io->first_reject = n_probs;
}

// ---------------------------------------------------------------- host side
struct DevRows {  // device copy of ragged rows
    DevBuf<double> data;
    DevBuf<int64_t> off;
    Rows view{nullptr, nullptr, 0};
    DevRows(const double* d, const int64_t* offsets, int n) {
        if (n < 0) throw_invalid("negative row count");
        if (n > 0 && (!d || !offsets)) throw_invalid("null probability rows");
        const int64_t total = n > 0 ? offsets[n] : 0;
        if (n > 0 && offsets[0] != 0) throw_invalid("row offsets must start at 0");
        for (int r = 0; r < n; ++r)
            if (offsets[r + 1] < offsets[r]) throw_invalid("row offsets must be non-decreasing");
        data.alloc(static_cast<size_t>(std::max<int64_t>(total, 1)));
        off.alloc(static_cast<size_t>(n) + 1);
        if (total > 0) CUDA_CHECK(cudaMemcpy(data.p, d, total * sizeof(double), cudaMemcpyHostToDevice));
        std::vector<int64_t> o(offsets ? offsets : nullptr, offsets ? offsets + n + 1 : nullptr);
        if (o.empty()) o.assign(1, 0);
        CUDA_CHECK(cudaMemcpy(off.p, o.data(), o.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        view = Rows{data.p, off.p, n};
    }
};

void raise(int err) {
    switch (err) {
        case 0: return;
        case kErrDegenerate: throw_runtime("degenerate distribution");                   // model.cpp:79
        case kErrResidualZero: throw_runtime("residual distribution is zero");           // verification.cpp:47,56
        case kErrDraftMassZero: throw_invalid("draft mass zero on emitted token");       // verification.cpp:21
        case kErrUncovered: throw_invalid("guided_output: reject position uncovered");   // verification.cpp:119,126
        default: throw_invalid("invalid argument");
    }
}

VerifyIO run_io(const std::function<void(VerifyIO*)>& launch) {
    DevBuf<VerifyIO> io(1);
    io.zero();
    launch(io.p);
    CUDA_LAUNCH_CHECK();
    VerifyIO h{};
    CUDA_CHECK(cudaMemcpy(&h, io.p, sizeof h, cudaMemcpyDeviceToHost));
    raise(h.err);
    return h;
}

}  // namespace

DeviceRng::DeviceRng(uint64_t seed, int device) : device_(device) {
    require_device(device);
    DeviceGuard gd(device);
    state_.alloc(1);
    rng_seed_kernel<<<1, 1>>>(state_.p, seed);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaDeviceSynchronize());
}
DeviceRng DeviceRng::derive(uint64_t seed, uint64_t round, uint64_t lane, int device) {  // rng.hpp:33-35
    return DeviceRng(derived_seed(seed, round, lane), device);
}
void DeviceRng::uniform(double* out, int n) {
    if (n < 0 || (n > 0 && !out)) throw_invalid("bad uniform request");
    if (n == 0) return;
    DeviceGuard gd(device_);
    DevBuf<double> d(n);
    rng_uniform_kernel<<<1, 1>>>(state_.p, d.p, n);
    CUDA_LAUNCH_CHECK();
    CUDA_CHECK(cudaMemcpy(out, d.p, n * sizeof(double), cudaMemcpyDeviceToHost));
}

double accept_prob(const double* p, int np, const double* q, int nq, int x, int device) {
    require_device(device);
    DeviceGuard gd(device);
    const int64_t op[2] = {0, np}, oq[2] = {0, nq};
    DevRows P(p, op, 1), Q(q, oq, 1);
    return run_io([&](VerifyIO* io) { accept_prob_kernel<<<1, 1>>>(P.view, Q.view, x, io); }).value;
}

int residual_sample(const double* p, int np, const double* q, int nq, DeviceRng& rng) {
    DeviceGuard gd(rng.device());
    const int64_t op[2] = {0, np}, oq[2] = {0, nq};
    DevRows P(p, op, 1), Q(q, oq, 1);
    return run_io([&](VerifyIO* io) { residual_kernel<<<1, 1>>>(P.view, Q.view, -1, rng.state(), io); }).token;
}

int residual_sample_point_mass(const double* p, int np, int x, DeviceRng& rng) {
    DeviceGuard gd(rng.device());
    const int64_t op[2] = {0, np};
    DevRows P(p, op, 1), Q(p, op, 1);
    if (x < 0) throw_invalid("token out of range");
    return run_io([&](VerifyIO* io) { residual_kernel<<<1, 1>>>(P.view, Q.view, x, rng.state(), io); }).token;
}

int verify_against_target(const int32_t* draft, int n_draft, const double* dprobs, const int64_t* doff, int n_dp,
                          const double* tprobs, const int64_t* toff, int n_tp, double temperature, DeviceRng& rng) {
    DeviceGuard gd(rng.device());
    if (n_draft < 0 || (n_draft > 0 && !draft)) throw_invalid("bad draft slice");
    DevBuf<int32_t> d(std::max(n_draft, 1));
    if (n_draft > 0) CUDA_CHECK(cudaMemcpy(d.p, draft, n_draft * 4, cudaMemcpyHostToDevice));
    DevRows DP(dprobs, doff, n_dp), TP(tprobs, toff, n_tp);
    return run_io([&](VerifyIO* io) {
               verify_kernel<<<1, 1>>>(d.p, n_draft, DP.view, TP.view, temperature, rng.state(), io);
           }).first_reject;
}

VerifyOutcome guided_output(const int32_t* draft, int n_draft, const double* dprobs, const int64_t* doff, int n_dp,
                            const int32_t* gtok, int n_gtok, const double* gprobs, const int64_t* goff, int n_gp,
                            int first_reject, double temperature, DeviceRng& rng) {
    DeviceGuard gd(rng.device());
    if (n_draft < 0 || (n_draft > 0 && !draft) || n_gtok < 0 || (n_gtok > 0 && !gtok))
        throw_invalid("bad token slice");
    DevBuf<int32_t> d(std::max(n_draft, 1)), gt(std::max(n_gtok, 1));
    if (n_draft > 0) CUDA_CHECK(cudaMemcpy(d.p, draft, n_draft * 4, cudaMemcpyHostToDevice));
    if (n_gtok > 0) CUDA_CHECK(cudaMemcpy(gt.p, gtok, n_gtok * 4, cudaMemcpyHostToDevice));
    DevRows DP(dprobs, doff, n_dp), GP(gprobs, goff, n_gp);
    const int cap = n_draft + n_gtok + 1;
    DevBuf<int32_t> out(cap);
    const VerifyIO h = run_io([&](VerifyIO* io) {
        guided_kernel<<<1, 1>>>(d.p, n_draft, DP.view, gt.p, n_gtok, GP.view, first_reject, temperature, rng.state(),
                                out.p, cap, io);
    });
    VerifyOutcome r;
    r.accepted_len = h.accepted_len;
    r.kind = h.kind;
    r.committed.resize(h.n_committed);
    if (h.n_committed > 0)
        CUDA_CHECK(cudaMemcpy(r.committed.data(), out.p, h.n_committed * 4, cudaMemcpyDeviceToHost));
    return r;
}

void tempered(const double* p, int n, double temperature, double* out, int device) {
    if (!(temperature > 0.0)) throw_invalid("tempered: temperature must be > 0");
    if (n < 0 || (n > 0 && (!p || !out))) throw_invalid("bad probability row");
    require_device(device);
    DeviceGuard gd(device);
    const int64_t op[2] = {0, n};
    DevRows P(p, op, 1);
    DevBuf<double> o(std::max(n, 1));
    run_io([&](VerifyIO* io) { tempered_kernel<<<1, 1>>>(P.view, temperature, o.p, io); });
    if (n > 0) CUDA_CHECK(cudaMemcpy(out, o.p, n * sizeof(double), cudaMemcpyDeviceToHost));
}

void argmax_rows(const double* probs, const int64_t* off, int n_rows, int32_t* out, int device) {
    if (n_rows <= 0) return;
    require_device(device);
    DeviceGuard gd(device);
    DevRows P(probs, off, n_rows);
    DevBuf<int32_t> o(n_rows);
    DevBuf<int> err(1);
    err.zero();
    argmax_rows_kernel<<<n_rows, kArgThreads>>>(P.view, o.p, err.p);
    CUDA_LAUNCH_CHECK();
    int h = 0;
    CUDA_CHECK(cudaMemcpy(&h, err.p, sizeof h, cudaMemcpyDeviceToHost));
    raise(h);
    CUDA_CHECK(cudaMemcpy(out, o.p, n_rows * 4, cudaMemcpyDeviceToHost));
}

int sample(const double* p, int n, double temperature, DeviceRng* rng, int device) {
    if (!(temperature >= 0.0)) throw_invalid("temperature must be >= 0");
    if (n < 0 || (n > 0 && !p)) throw_invalid("bad probability row");
    if (temperature == 0.0) {
        const int64_t op[2] = {0, n};
        int32_t t = 0;
        argmax_rows(p, op, 1, &t, device);
        return t;
    }
    if (!rng) throw_invalid("sample: an Rng is required at temperature > 0");
    DeviceGuard gd(rng->device());
    const int64_t op[2] = {0, n};
    DevRows P(p, op, 1);
    DevBuf<double> eff(std::max(n, 1));
    return run_io([&](VerifyIO* io) { sample_kernel<<<1, 1>>>(P.view, temperature, rng->state(), eff.p, io); }).token;
}

namespace {
// accept_with_model over rows already on the device (D) whose offsets are off_host
AcceptOut accept_impl(const Rows& D, const int64_t* off_host, int n_rows, const int32_t* cands, int c,
                      double temperature, DeviceRng* rng, bool want_probs) {
    if (c < 0 || (c > 0 && !cands)) throw_invalid("bad candidate slice");
    if (n_rows != c + 1) throw_invalid("accept_with_model: need |cands|+1 distributions");  // speculation.cpp:11
    if (!(temperature >= 0.0)) throw_invalid("temperature must be >= 0");
    if (temperature != 0.0 && !rng) throw_invalid("accept_with_model: an Rng is required at temperature > 0");
    const int64_t total = off_host[n_rows];
    DevBuf<double> E(static_cast<size_t>(temperature != 0.0 ? std::max<int64_t>(total, 1) : 1));
    DevBuf<int32_t> cd(std::max(c, 1)), em(c + 1);
    if (c > 0) CUDA_CHECK(cudaMemcpy(cd.p, cands, c * 4, cudaMemcpyHostToDevice));
    const VerifyIO h = run_io([&](VerifyIO* io) {
        accept_model_kernel<<<1, 1>>>(D, cd.p, c, temperature, rng ? rng->state() : nullptr, E.p, em.p, io);
    });
    AcceptOut r;
    r.matched_len = h.accepted_len;
    r.emitted.resize(h.n_committed);
    CUDA_CHECK(cudaMemcpy(r.emitted.data(), em.p, h.n_committed * 4, cudaMemcpyDeviceToHost));
    r.n_probs = h.first_reject;
    if (want_probs) {
        const int64_t len = off_host[r.n_probs];
        r.probs.resize(static_cast<size_t>(len));
        if (len > 0)
            CUDA_CHECK(cudaMemcpy(r.probs.data(), temperature == 0.0 ? D.data : E.p, len * sizeof(double),
                                  cudaMemcpyDeviceToHost));
    }
    return r;
}
}  // namespace

AcceptOut accept_with_model(const double* dists, const int64_t* off, int n_rows, const int32_t* cands, int c,
                            double temperature, DeviceRng* rng, int device, bool want_probs) {
    if (n_rows != c + 1) throw_invalid("accept_with_model: need |cands|+1 distributions");  // speculation.cpp:11
    const int dev = rng ? rng->device() : device;
    require_device(dev);
    DeviceGuard gd(dev);
    DevRows D(dists, off, n_rows);
    return accept_impl(D.view, off, n_rows, cands, c, temperature, rng, want_probs);
}

AcceptOut accept_with_model_dev(const double* dists_dev, int vocab, int n_rows, const int32_t* cands, int c,
                                double temperature, DeviceRng* rng, bool want_probs) {
    std::vector<int64_t> off(static_cast<size_t>(n_rows) + 1);
    for (int r = 0; r <= n_rows; ++r) off[r] = static_cast<int64_t>(r) * vocab;
    DevBuf<int64_t> doff(off.size());
    CUDA_CHECK(cudaMemcpy(doff.p, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    return accept_impl(Rows{dists_dev, doff.p, n_rows}, off.data(), n_rows, cands, c, temperature, rng, want_probs);
}

}  // namespace dbl
