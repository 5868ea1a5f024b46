// K2' — the order-m probability-table model of config 1 on the device (specpar::TableModel,
// model.hpp:18-25).  One warp per row: BOS-padded window (window_of, model.cpp:13-21) -> open-
// addressing hash probe -> fp64 argmax with the reference's lowest-id tie-break (model.cpp:70-81).
#include <vector>

#include "model.cuh"
#include "table_model.cuh"

namespace dbl {

namespace {

__host__ __device__ inline unsigned long long mix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d49bb133111ebull;
    return x ^ (x >> 31);
}
__host__ __device__ inline unsigned long long window_hash(const int32_t* w, int order) {
    unsigned long long h = 0xcbf29ce484222325ull;
    for (int i = 0; i < order; ++i) h = (h ^ static_cast<uint32_t>(w[i])) * 0x100000001b3ull;
    return mix64(h);
}

struct TableDev {
    const int32_t* windows;
    const int32_t* slots;
    const double* probs;
    const double* fallback;
    int order, vocab, cap_mask;
};

// rows p in [row_from, L+c): argmax of the distribution after buf[0..p]
__global__ void table_forward_kernel(TableDev t, const int32_t* __restrict__ buf, LaneState* lane,
                                     int32_t* __restrict__ argmax, float* __restrict__ probs_out,
                                     double* __restrict__ dist_out) {
    const int L = lane->L, c = lane->c;
    const int row_from = lane->row0;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, ln = threadIdx.x & 31;
    const int p = row_from + warp;
    if (p < L + c) {
        int w[kMaxTableOrder];
        for (int i = 0; i < t.order; ++i) {
            const int src = p - (t.order - 1) + i;
            w[i] = src >= 0 ? buf[src] : 0;  // kBosToken = 0, types.hpp:15
        }
        int row = -1;
        if (ln == 0) {
            unsigned long long h = window_hash(w, t.order) & static_cast<unsigned long long>(t.cap_mask);
            for (;;) {
                const int r = t.slots[h];
                if (r < 0) break;
                bool eq = true;
                for (int i = 0; i < t.order; ++i) eq &= t.windows[static_cast<long>(r) * t.order + i] == w[i];
                if (eq) { row = r; break; }
                h = (h + 1) & static_cast<unsigned long long>(t.cap_mask);
            }
        }
        row = __shfl_sync(0xffffffffu, row, 0);
        const double* pr = row >= 0 ? t.probs + static_cast<long>(row) * t.vocab : t.fallback;
        double best = -1.0;
        int bi = 0;
        for (int v = ln; v < t.vocab; v += 32) {
            const double x = pr[v];
            if (x > best) { best = x; bi = v; }  // strict: lowest id within the lane's stride
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (ln == 0) {
            if (best <= 0.0) { argmax[p] = -1; lane->error = 1; }
            else argmax[p] = bi;
        }
        if (probs_out)
            for (int v = ln; v < t.vocab; v += 32)
                probs_out[static_cast<long>(p - row_from) * t.vocab + v] = static_cast<float>(pr[v]);
        if (dist_out)  // the ProbVector itself (row_for, model.cpp:23-35): exact fp64 copy
            for (int v = ln; v < t.vocab; v += 32) dist_out[static_cast<long>(p - row_from) * t.vocab + v] = pr[v];
    }
}

__global__ void table_finish_kernel(LaneState* lane) {
    lane->start = lane->row0;
    lane->kv_len = lane->L + lane->c;
}

}  // namespace

TableModel::TableModel(int order, int vocab, int64_t n_rows, const int32_t* windows,
                       const double* probs, const double* fallback, int device)
    : device_(device), order_(order), vocab_(vocab), n_rows_(n_rows) {
    if (order < 1 || order > kMaxTableOrder) throw_invalid("table order out of range");
    if (vocab < 1) throw_invalid("table vocab must be >= 1");
    if (n_rows < 0) throw_invalid("negative row count");
    require_device(device);
    DeviceGuard g(device);
    long cap = 64;
    while (cap < 2 * n_rows + 2) cap *= 2;
    std::vector<int32_t> slots(cap, -1);
    for (int64_t r = 0; r < n_rows; ++r) {
        unsigned long long h = window_hash(windows + r * order, order) & static_cast<unsigned long long>(cap - 1);
        while (slots[h] >= 0) {
            bool eq = true;
            for (int i = 0; i < order; ++i) eq &= windows[slots[h] * order + i] == windows[r * order + i];
            if (eq) throw_invalid("duplicate table window");
            h = (h + 1) & static_cast<unsigned long long>(cap - 1);
        }
        slots[h] = static_cast<int32_t>(r);
    }
    cap_mask_ = static_cast<int>(cap - 1);
    windows_.alloc(std::max<int64_t>(n_rows * order, 1));
    slots_.alloc(cap);
    probs_.alloc(std::max<int64_t>(n_rows * vocab, 1));
    fallback_.alloc(vocab);
    if (n_rows) {
        CUDA_CHECK(cudaMemcpy(windows_.p, windows, n_rows * order * 4, cudaMemcpyHostToDevice));
        CUDA_CHECK(cudaMemcpy(probs_.p, probs, n_rows * vocab * 8, cudaMemcpyHostToDevice));
    }
    CUDA_CHECK(cudaMemcpy(slots_.p, slots.data(), cap * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(fallback_.p, fallback, vocab * 8, cudaMemcpyHostToDevice));
}

void TableModel::launch(Lane& lane, int max_tokens, float* probs_out, double* dist_out, cudaStream_t s) {
    TableDev t{windows_.p, slots_.p, probs_.p, fallback_.p, order_, vocab_, cap_mask_};
    const int rows = std::max(max_tokens, 1);
    const int threads = 256, warps_per_block = threads / 32;
    table_forward_kernel<<<(rows + warps_per_block - 1) / warps_per_block, threads, 0, s>>>(
        t, lane.buf.p, lane.state, lane.argmax.p, probs_out, dist_out);
    CUDA_LAUNCH_CHECK();
    table_finish_kernel<<<1, 1, 0, s>>>(lane.state);
    CUDA_LAUNCH_CHECK();
}

void TableModel::forward(Lane& lane, int max_tokens, cudaStream_t s) {
    launch(lane, max_tokens, nullptr, nullptr, s);
}

void TableModel::logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) {
    launch(lane, max_tokens, out_dev, nullptr, s);
}

void TableModel::dists(Lane& lane, int max_tokens, int, double* out_dev, cudaStream_t s) {
    launch(lane, max_tokens, nullptr, out_dev, s);
}

}  // namespace dbl
