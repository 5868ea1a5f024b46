// K3 — greedy acceptance kernels.  They consume the per-position argmax rows a forward produced and
// advance the lane cursor on the device, so the draft's gamma chain never returns to the host.
//   draft segment : accept_with_model (speculation.cpp:7-52) + the chain append of iterative_draft
//                   (speculation.cpp:76-84); KV commit = kv_len := new L - 1 (nothing moves)
//   target round  : verify_against_target greedy (verification.cpp:60-78) on the speculative tail +
//                   accept_with_model on the target's retrieved candidates (pipeline.cpp:60-68)
// One warp each: the first mismatch is a ballot over 32 positions per round trip (the reference's
// sequential scans, same result).  Results land directly in mapped pinned host memory (RoundResult).
#include "accept.cuh"

namespace dbl {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// first i in [0, n) with bad(i), else n — one warp, 32 positions per round trip (ballot + ffs)
template <class F>
__device__ __forceinline__ int warp_first(int n, F bad) {
    const int ln = threadIdx.x & 31;
    for (int b = 0; b < n; b += 32) {
        const int i = b + ln;
        const unsigned m = __ballot_sync(kFull, i < n && bad(i));
        if (m) return b + __ffs(m) - 1;
    }
    return n;
}

__global__ void draft_accept_kernel(const int32_t* __restrict__ argmax, int32_t* buf, LaneState* lane,
                                    int vocab, RoundResult* rr, int seg) {
    const int ln = threadIdx.x;
    const int L = lane->L, c = lane->c;
    // accept while cands[s] is in [0, V) (speculation.cpp:19) and equals the row's argmax
    const int s = warp_first(c, [&](int i) {
        const int cand = buf[L + i];
        return cand < 0 || cand >= vocab || cand != argmax[L - 1 + i];
    });
    const int tok = argmax[L - 1 + s];  // correction or continuation (greedy: argmax either way)
    const int base = L - rr->draft_L0;
    const bool fits = base + s + 1 <= kMaxRoundTokens;
    if (fits)
        for (int i = ln; i <= s; i += 32) rr->draft_tokens[base + i] = i < s ? buf[L + i] : tok;
    __syncwarp();
    if (ln != 0) return;
    if (tok < 0) { lane->error = 1; rr->draft_error = 1; }
    if (!fits) rr->draft_error = 2;
    buf[L + s] = tok;
    rr->segs[seg] = SegRecord{s, s + 1, lane->src, lane->order};
    rr->n_segs = seg + 1;
    const int Ln = L + s + 1;
    rr->draft_L = Ln;
    lane->L = Ln;
    lane->c = 0;
    lane->kv_len = Ln - 1;  // positions < L+s saw the final tokens; L+s did not
    lane->row0 = Ln - 1;
    lane->src = DBL_SRC_MISS;
    lane->order = 0;
}

__global__ void target_accept_kernel(const int32_t* __restrict__ argmax, const int32_t* __restrict__ buf,
                                     LaneState* lane, int vocab, int n_committed, RoundResult* rr) {
    const int ln = threadIdx.x;
    const int L = lane->L, c = lane->c;
    const int n_spec = L - n_committed;
    if (c + 1 > kMaxRoundTokens) {  // host-validated (depth < kMaxRoundTokens); never write past the record
        if (ln == 0) {
            lane->error = 2;
            rr->target_error = 2;
            rr->ext_c = 0;
        }
        return;
    }
    // pre-verify of the speculative tail (verification.cpp:60-78, greedy): the first mismatch
    const int k = warp_first(n_spec, [&](int i) { return buf[n_committed + i] != argmax[n_committed - 1 + i]; });
    const int rej = k < n_spec ? k : -1;
    // the target's own retrieved candidates (accept_with_model, pipeline.cpp:60-68)
    const int s = warp_first(c, [&](int i) {
        const int cand = buf[L + i];
        return cand < 0 || cand >= vocab || cand != argmax[L - 1 + i];
    });
    const int last = argmax[L - 1 + s];
    for (int i = ln; i < c; i += 32) {
        const int cand = buf[L + i];
        rr->ext_cands[i] = cand;
        if (i < s) rr->ext_emitted[i] = cand;
    }
    // degenerate rows among those consumed: the verified prefix, the correction, the emitted token
    const int nv = rej >= 0 ? rej : n_spec;
    const bool bad_row = warp_first(nv, [&](int i) { return argmax[n_committed - 1 + i] < 0; }) < nv;
    __syncwarp();
    if (ln != 0) return;
    const int corr = rej >= 0 ? argmax[n_committed - 1 + rej] : -1;
    rr->tgt_rej = rej;
    rr->tgt_correction = corr;
    rr->ext_emitted[s] = last;
    rr->ext_matched = s;
    rr->ext_source = lane->src;
    rr->ext_order = lane->order;
    rr->ext_c = c;
    if (last < 0 || (rej >= 0 && corr < 0) || bad_row) { lane->error = 1; rr->target_error = 1; }
    lane->kv_len = L + c;
}

}  // namespace

void launch_draft_accept(Lane& lane, RoundResult* rr_dev, int seg, cudaStream_t s) {
    draft_accept_kernel<<<1, 32, 0, s>>>(lane.argmax.p, lane.buf.p, lane.state, lane.model.vocab(),
                                         rr_dev, seg);
    CUDA_LAUNCH_CHECK();
}

void launch_target_accept(Lane& lane, int n_committed, RoundResult* rr_dev, cudaStream_t s) {
    target_accept_kernel<<<1, 32, 0, s>>>(lane.argmax.p, lane.buf.p, lane.state, lane.model.vocab(),
                                          n_committed, rr_dev);
    CUDA_LAUNCH_CHECK();
}

}  // namespace dbl
