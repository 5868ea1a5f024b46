// Device-resident hierarchical n-gram datastore (replaces specpar::HierarchicalDatastore,
// datastore.hpp:19-95).
//
// HBM layout, per layer (prior / dynamic / rejected), append-only:
//   tokens[n_tokens]   every stored sequence back to back (int32)
//   seq_of[n_tokens]   owning sequence id of each token  (coalesced scan key)
//   seq_start/len/step per sequence (the Occurrence fields, datastore.hpp:11-15)
// plus, for a bulk-loaded layer (build_prior / a dstore-v1 prior: the large, static one), an n-gram
// index over its first idx_tokens tokens — the device form of the reference's std::map n-gram ->
// occurrence list (datastore.cpp:9-20):
//   idx_occ[E]         every indexed occurrence (sequence, end position p of an n-gram, n = 1..order,
//                      whose sequence continues after p), sorted by a 64-bit hash of (n, the n tokens)
//   idx_table          open-addressing table: hash -> its run [start, start + count) in idx_occ
// A lookup probes the table for the context suffix at each order (one round trip), scans only that
// run (hash collisions are rejected by comparing the tokens) and reduces the reference's 4-key
// lexicographic max (step, avail, seq_id, end_pos) (datastore.cpp:49-71).  Tokens past idx_tokens
// (the dynamic / rejected layers, and anything appended to an indexed layer later) are scanned: one
// CTA-cooperative pass evaluates every position against the context suffix for all orders at once.
// The PLD fallback (datastore.cpp:109-128) is a scan over the context.  Inserts are O(len) appends,
// which is what makes the per-round datastore update (pipeline.cpp:146-184) a single tiny kernel.
#pragma once
#include <memory>
#include <utility>
#include <vector>

#include "common.cuh"
#include "lane.cuh"

namespace dbl {

struct LayerDesc {
    int32_t* tokens;
    int32_t* seq_of;
    int32_t* seq_start;
    int32_t* seq_len;
    int64_t* seq_step;
    int32_t n_tokens;
    int32_t n_seqs;
    int32_t max_order;
    int32_t idx_tokens;  // tokens [0, idx_tokens) are covered by the n-gram index (0: none)
    const struct IdxSlot* idx_table;     // [idx_mask + 1] hash -> run (key 0 = empty slot)
    const unsigned long long* idx_occ;   // [E] occurrences (seq << 32 | end position), grouped by hash
    uint32_t idx_mask;
    int32_t idx_order;                   // orders 1..idx_order are indexed
};
struct alignas(16) IdxSlot {  // one 16-byte load per probe
    unsigned long long key;
    uint32_t start, count;   // the n-gram's run [start, start + count) in idx_occ
};

struct StoreDesc {  // lives in device memory; kernels read counts from here (graph-safe)
    LayerDesc layer[3];
    int32_t max_order;
    int32_t rejected_enabled;
    unsigned long long stats[6];  // lookups, prior, dynamic, rejected, fallback, misses
};

class DeviceStore {
  public:
    DeviceStore(int max_order, int depth, int device);
    ~DeviceStore();
    int device() const { return device_; }
    int max_order() const { return max_order_; }
    int depth() const { return depth_; }
    long step() const { return step_; }
    void set_step(long s) { step_ = s; }
    bool rejected_enabled() const { return rejected_enabled_; }
    void set_rejected_enabled(bool on, cudaStream_t s);
    void set_layer_order(int layer, int order, cudaStream_t s);

    // append-only insert (NGramIndex::insert): enqueued on stream s, tokens copied immediately
    void insert(int layer, const int32_t* tokens, int n, long step, cudaStream_t s);
    void record(int layer, const int32_t* tokens, int n, cudaStream_t s) {  // datastore.cpp:134-142
        if (n <= 0) return;
        insert(layer, tokens, n, step_++, s);
    }
    void clear_layer(int layer, cudaStream_t s);
    // layer := n_seqs sequences (offsets into toks) with steps 0..n-1 (build_prior, datastore.cpp:149-159)
    void load_layer(int layer, int max_order, const int64_t* off, const int32_t* toks, int n_seqs, cudaStream_t s);
    // (re)build the n-gram index over the layer's current tokens (load_layer does this for the prior)
    void build_index(int layer, cudaStream_t s);
    int64_t index_entries(int layer) const;
    std::unique_ptr<DeviceStore> clone() const { return clone_to(device_); }
    std::unique_ptr<DeviceStore> clone_to(int device) const;  // a replica on another GPU (draft-side lookups)
    void add_stats(const int64_t delta[6], cudaStream_t s);   // fold a replica's lookup counts in
    void flush_session(cudaStream_t s) { clear_layer(1, s); clear_layer(2, s); }

    // one lookup for a lane: ctx = buf[0, lane.L); candidates -> buf[L, L+c), lane.c/src/order
    void lookup_lane(int32_t* buf, LaneState* lane, int d, cudaStream_t s) const;
    // batch of independent host queries (tests / throughput)
    void lookup_batch(int n_q, const int64_t* offsets, const int32_t* toks, const int32_t* depths,
                      int d_cap, int32_t* out_cands, int32_t* out_n, int32_t* out_src,
                      int32_t* out_order, cudaStream_t s);
    double profile_lookup(const int32_t* ctx, int L, int d, int iters);  // us per lookup (device)
    void stats(int64_t out[6], cudaStream_t s) const;
    void layer_info(int layer, int64_t* n_seqs, int64_t* n_tokens, int64_t* occ) const;
    void layer_read(int layer, int32_t* toks, int64_t tok_cap, int32_t* lens, int64_t* steps,
                    int64_t seq_cap, cudaStream_t s) const;
    StoreDesc* desc_dev() const { return desc_dev_; }

  private:
    struct HostLayer {
        int32_t n_tokens = 0, n_seqs = 0, tok_cap = 0, seq_cap = 0, max_order = 3;
        std::vector<int32_t> lens;  // host mirror of sequence lengths (occurrence_count)
        DevBuf<int32_t> tokens, seq_of, seq_start, seq_len;
        DevBuf<int64_t> seq_step;
        // n-gram index over tokens [0, idx_tokens) (build_index)
        int32_t idx_tokens = 0, idx_order = 0;
        uint32_t idx_mask = 0;
        DevBuf<IdxSlot> idx_table;
        DevBuf<unsigned long long> idx_occ;
    };
    LayerDesc desc_of(const HostLayer& h) const;
    void grow(int layer, int need_tok, int need_seq, cudaStream_t s);
    void push_desc(cudaStream_t s);
    int device_, max_order_, depth_;
    long step_ = 0;
    bool rejected_enabled_ = true;
    HostLayer layers_[3];
    StoreDesc* desc_dev_ = nullptr;
    struct Staging {  // mapped pinned ring for insert payloads + the last append per stream using it
        PinBuf<int32_t> buf;
        std::vector<std::pair<cudaStream_t, cudaEvent_t>> pend;
        void drain();
        void mark(cudaStream_t s);
    };
    Staging staging_[2];
    int staging_cur_ = 0;
    size_t staging_at_ = 0;
};

}  // namespace dbl
