// Device-resident hierarchical n-gram datastore (replaces specpar::HierarchicalDatastore,
// datastore.hpp:19-95).
//
// HBM layout, per layer (prior / dynamic / rejected), append-only:
//   tokens[n_tokens]   every stored sequence back to back (int32)
//   seq_of[n_tokens]   owning sequence id of each token  (coalesced scan key)
//   seq_start/len/step per sequence (the Occurrence fields, datastore.hpp:11-15)
// The reference's std::map n-gram -> occurrence list (datastore.cpp:9-20) is implicit: an occurrence
// of an n-gram is any position whose last n tokens (within its sequence) equal it.  A lookup is a
// single CTA-cooperative scan that evaluates every position against the context suffix for all
// orders at once and reduces the reference's 4-key lexicographic max (step, avail, seq_id, end_pos)
// (datastore.cpp:49-71) per (layer, order); the PLD fallback (datastore.cpp:109-128) is a second scan
// over the context.  Inserts are O(len) appends — no index maintenance — which is what makes the
// per-round datastore update (pipeline.cpp:146-184) a single tiny kernel.
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
    int32_t pad;
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
    std::unique_ptr<DeviceStore> clone() const;
    void flush_session(cudaStream_t s) { clear_layer(1, s); clear_layer(2, s); }

    // one lookup for a lane: ctx = buf[0, lane.L); candidates -> buf[L, L+c), lane.c/src/order
    void lookup_lane(int32_t* buf, LaneState* lane, int d, cudaStream_t s) const;
    // batch of independent host queries (tests / throughput)
    void lookup_batch(int n_q, const int64_t* offsets, const int32_t* toks, const int32_t* depths,
                      int d_cap, int32_t* out_cands, int32_t* out_n, int32_t* out_src,
                      int32_t* out_order, cudaStream_t s);
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
    };
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
