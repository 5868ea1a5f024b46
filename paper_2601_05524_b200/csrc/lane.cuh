// Per-model decode "lane": the token buffer a model reads and the device-resident cursor the
// retrieval, forward and acceptance kernels advance without host round trips.
//
// buf[0, L)        : the model's working context (committed ⊕ speculative ⊕ emitted so far)
// buf[L, L+c)      : candidates written in place by the lookup kernel (datastore.cpp:73-78 /
//                    :118-124 continuation), so a forward reads buf[start, L+c) contiguously
// rows             : argmax[p] = argmax of the next-token distribution after buf[0..p]
//                    (forward_batch row semantics, model.cpp:37-53), for p in [start, L+c)
// kv_len           : positions [0, kv_len) hold valid KV (transformers); a forward processes
//                    [min(kv_len, row0), L+c) — the "rollback-free" commit is just kv_len.
#pragma once
#include <cstdint>

namespace dbl {

struct LaneState {
    int32_t L;        // context length
    int32_t c;        // candidates at buf[L, L+c)
    int32_t kv_len;   // valid KV prefix
    int32_t row0;     // first position whose row is consumed
    int32_t src;      // last lookup source (dbl_source)
    int32_t order;    // last lookup matched order
    int32_t start;    // first position processed by the last forward
    int32_t error;    // sticky device error (1 = degenerate distribution, 2 = capacity)
};

// Draft-chain segment record (RetrievalResult, speculation.hpp:12-17, greedy: probs omitted)
struct SegRecord {
    int32_t matched;  // matched_len
    int32_t n_emit;   // matched_len + 1
    int32_t source;   // LookupSource of this segment's lookup (Miss when retrieval is off)
    int32_t order;
};

// Everything the host orchestrator needs after a round, written by kernels straight into mapped
// pinned host memory (no D2H copies on the critical path).
constexpr int kMaxSegs = 64;
constexpr int kMaxRoundTokens = 4096;
struct RoundResult {
    // draft lane
    int32_t draft_L0, draft_L;          // context length before / after the chain
    int32_t n_segs;
    SegRecord segs[kMaxSegs];
    int32_t draft_error;
    // target lane
    int32_t tgt_rej;                     // first rejected speculative index, -1 if none
    int32_t tgt_correction;              // argmax at the rejected position
    int32_t ext_matched, ext_source, ext_order, ext_c;
    int32_t ext_emitted[kMaxRoundTokens];  // ext.emitted (matched cands + 1)
    int32_t ext_cands[kMaxRoundTokens];    // all candidates the target scored (KV mirror)
    int32_t target_error;
    int32_t draft_tokens[kMaxRoundTokens]; // the chain (buf[draft_L0, draft_L))
};

}  // namespace dbl
