// K3 — greedy acceptance kernels.  They consume the per-position argmax rows a forward produced and
// advance the lane cursor on the device, so the draft's gamma chain never returns to the host.
//   draft segment : accept_with_model (speculation.cpp:7-52) + the chain append of iterative_draft
//                   (speculation.cpp:76-84); KV commit = kv_len := new L - 1 (nothing moves)
//   target round  : verify_against_target greedy (verification.cpp:60-78) on the speculative tail +
//                   accept_with_model on the target's retrieved candidates (pipeline.cpp:60-68)
// Results land directly in mapped pinned host memory (RoundResult).
#include "accept.cuh"

namespace dbl {

namespace {

__global__ void draft_accept_kernel(const int32_t* __restrict__ argmax, int32_t* buf, LaneState* lane,
                                    int vocab, RoundResult* rr, int seg) {
    if (threadIdx.x != 0) return;
    const int L = lane->L, c = lane->c;
    int s = 0;
    while (s < c) {
        const int cand = buf[L + s];
        if (cand < 0 || cand >= vocab) break;  // speculation.cpp:19
        if (cand != argmax[L - 1 + s]) break;
        ++s;
    }
    const int tok = argmax[L - 1 + s];  // correction or continuation (greedy: argmax either way)
    if (tok < 0) { lane->error = 1; rr->draft_error = 1; }
    buf[L + s] = tok;
    const int base = L - rr->draft_L0;
    if (base + s + 1 <= kMaxRoundTokens)
        for (int i = 0; i <= s; ++i) rr->draft_tokens[base + i] = buf[L + i];
    else
        rr->draft_error = 2;
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
    if (threadIdx.x != 0) return;
    const int L = lane->L, c = lane->c;
    const int n_spec = L - n_committed;
    if (c + 1 > kMaxRoundTokens) {  // host-validated (depth < kMaxRoundTokens); never write past the record
        lane->error = 2;
        rr->target_error = 2;
        rr->ext_c = 0;
        return;
    }
    int rej = -1;
    for (int k = 0; k < n_spec; ++k) {
        if (buf[n_committed + k] != argmax[n_committed - 1 + k]) { rej = k; break; }
    }
    rr->tgt_rej = rej;
    rr->tgt_correction = rej >= 0 ? argmax[n_committed - 1 + rej] : -1;
    int s = 0;
    while (s < c) {
        const int cand = buf[L + s];
        if (cand < 0 || cand >= vocab) break;
        if (cand != argmax[L - 1 + s]) break;
        ++s;
    }
    for (int i = 0; i < s; ++i) rr->ext_emitted[i] = buf[L + i];
    rr->ext_emitted[s] = argmax[L - 1 + s];
    for (int i = 0; i < c; ++i) rr->ext_cands[i] = buf[L + i];
    rr->ext_matched = s;
    rr->ext_source = lane->src;
    rr->ext_order = lane->order;
    rr->ext_c = c;
    bool bad = argmax[L - 1 + s] < 0 || (rej >= 0 && rr->tgt_correction < 0);
    for (int k = 0; k < (rej >= 0 ? rej : n_spec); ++k) bad |= argmax[n_committed - 1 + k] < 0;
    if (bad) { lane->error = 1; rr->target_error = 1; }
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
