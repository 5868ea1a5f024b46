// Host orchestrator of the device decode loop (replaces specpar::run / run_round / finish_round,
// pipeline.cpp:15-323; run_vanilla_ar / run_serial_sd, harness.cpp:233-369).
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "model.cuh"
#include "store.cuh"
#include "verify.cuh"

namespace dbl {

constexpr int kMaxBatchSeqs = 16;  // sequences per batched forward (FwdBatch, fwd.cuh)

struct Trace {  // RoundTrace, pipeline.hpp:57-71
    long round = 0;
    std::string mode;
    int pending = 0, draft_len = 0;
    std::vector<int> draft_matched;
    int target_matched = -1;
    std::string target_source;
    int accepted_pending = 0;
    bool pending_reject = false, rejected = false;
    int committed_count = 0;
    std::string kind;
    double clock_delta = 0.0;
};

struct RunOutput {
    std::vector<int32_t> output;
    std::vector<Trace> traces;
    dbl_run_metrics metrics{};
    // Decision log (argmax rows the loop consumed), per round:
    //   n_segs, {matched, emitted[matched+1]} x n_segs, n_spec, rej, correction, ext_matched,
    //   ext_emitted[ext_matched+1]
    // It lets the reference loop be replayed on the host with the forward excluded (bench.py).
    std::vector<int32_t> log;
};

std::string traces_to_jsonl(const std::vector<Trace>& traces);
void compute_metrics(const std::vector<Trace>& traces, double t_target, dbl_run_metrics* m);

RunOutput run_double(Model& draft, Model& target, DeviceStore& store, const int32_t* prompt,
                     int n_prompt, int max_new, const dbl_pipeline_options& o);
// run for up to kMaxBatchSeqs independent sequences (one datastore each) with batched forwards
std::vector<RunOutput> run_double_multi(Model& draft, Model& target, const std::vector<DeviceStore*>& stores,
                                        const std::vector<std::vector<int32_t>>& prompts, int max_new,
                                        const dbl_pipeline_options& o);
RunOutput run_ar(Model& target, const int32_t* prompt, int n_prompt, int max_new, double t_target,
                 double temperature, uint64_t seed);
// run_vanilla_ar for up to kMaxBatchSeqs sequences in lockstep, one batched forward per step
std::vector<RunOutput> run_ar_batch(Model& target, const std::vector<std::vector<int32_t>>& prompts, int max_new,
                                    double t_target, double* device_ms, long long* launches);
RunOutput run_serial_sd(Model& draft, Model& target, DeviceStore& store, const int32_t* prompt,
                        int n_prompt, int max_new, const dbl_pipeline_options& o, bool use_retrieval);

// PipelineState (pipeline.hpp:46-55) on the host side of the run_round boundary
struct HostPipelineState {
    std::vector<int32_t> committed, speculative;
    long n_spec_probs = 0;                  // |spec_probs| (check_state compares it with |speculative|)
    const double* spec_probs_in = nullptr;  // T > 0: |speculative| x vocab rows (host), or null = the
                                            // session's own device rows from its previous round
    int mode = 0;                           // Mode::PreVerify 0 / PostVerify 1
    int prev_tokens = 0;
    long round = 0;
    double clock = 0.0;                     // SimClock::now
    long last_committed_len = 0;
};

// run_round (pipeline.cpp:223-262) one call at a time: the draft/target lanes (KV) persist in the
// session and are re-synchronised with whatever state is passed in (longest common prefix).
class RoundSession {
  public:
    RoundSession(Model& draft, Model& target);
    ~RoundSession();
    // one round: st advanced in place (committed, speculative, mode, prev_tokens, round, clock,
    // last_committed_len); spec_probs_out (T > 0) receives the new speculative tail's rows
    Trace run_round(HostPipelineState& st, DeviceStore& store, const dbl_pipeline_options& o,
                    std::vector<double>* spec_probs_out);

  private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

// forward of `rows` tokens after a ctx_len context, timed (out[8], see decoder.cu)
void profile_forward(Model& m, int ctx_len, int rows, int iters, double* out);

// forward_batch as a stateless call (fresh lane / KV): argmax rows (c+1) and optionally logits
void forward_stateless(Model& m, const int32_t* ctx, int L, const int32_t* cands, int c,
                       int32_t* out_argmax, float* out_logits, double* out_dists = nullptr,
                       DevBuf<double>* keep_dists = nullptr);

struct RetrievalOut {  // RetrievalResult (speculation.hpp:12-17)
    std::vector<int32_t> emitted;
    int matched_len = 0;
    int source = DBL_SRC_MISS;
    int n_probs = 0;            // rows in probs (each vocab long)
    std::vector<double> probs;  // filled when asked
};
// retrieval_forward (speculation.cpp:54-66); rng may be null when temperature == 0
RetrievalOut retrieval_forward(Model& m, DeviceStore* st, const int32_t* ctx, int L, int depth, double temperature,
                               DeviceRng* rng, bool use_retrieval, bool want_probs);

}  // namespace dbl
