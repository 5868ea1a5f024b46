/* double_b200.h — the C-ABI drop-in boundary of the B200-native DOUBLE decode loop.
 *
 * The reference (arXiv 2601.05524 artifact, /root/reference/proj) exposes its decode path as C++ free
 * functions and structs in proj/include/specpar/*.hpp.  This header is the thin C layer the C++ host
 * code (include/double_b200.hpp, namespace specpar) calls; every entry point below names the
 * reference interface it replaces.  Conventions:
 *   - plain pointers + sizes, no C++ or torch types; host buffers unless a name says "_dev";
 *   - every call returns a dbl_status; dbl_last_error() returns the thread's last message;
 *   - errors map 1:1 onto the reference's exception types (std::invalid_argument ->
 *     DBL_INVALID_ARGUMENT, std::runtime_error -> DBL_RUNTIME_ERROR, std::logic_error ->
 *     DBL_LOGIC_ERROR), so the C++ shim rethrows the same types (pipeline.cpp:18-22, 210-217);
 *   - there is no CPU fallback: without a usable sm_100 device every compute entry point fails with
 *     DBL_CUDA_ERROR.
 */
#ifndef DOUBLE_B200_H
#define DOUBLE_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
    DBL_OK = 0,
    DBL_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    DBL_RUNTIME_ERROR = 2,    /* std::runtime_error    */
    DBL_LOGIC_ERROR = 3,      /* std::logic_error      */
    DBL_CUDA_ERROR = 4,
    DBL_NCCL_ERROR = 5
} dbl_status;

/* LookupSource (datastore.hpp:29) — same order */
typedef enum { DBL_SRC_PRIOR = 0, DBL_SRC_DYNAMIC = 1, DBL_SRC_REJECTED = 2, DBL_SRC_CONTEXT = 3, DBL_SRC_MISS = 4 } dbl_source;
/* datastore layers */
typedef enum { DBL_LAYER_PRIOR = 0, DBL_LAYER_DYNAMIC = 1, DBL_LAYER_REJECTED = 2 } dbl_layer;

typedef struct dbl_store_s* dbl_store_t;     /* device-resident HierarchicalDatastore */
typedef struct dbl_model_s* dbl_model_t;     /* device model: table (config 1) or transformer */
typedef struct dbl_rng_s* dbl_rng_t;         /* specpar::Rng: mt19937_64 stream resident on the device */

const char* dbl_last_error(void);
int dbl_version(void);
/* 1 when a CUDA device of compute capability 10.x is visible and the kernels load */
int dbl_device_ok(void);

/* ===================================================================== datastore
 * Replaces specpar::HierarchicalDatastore / NGramIndex (datastore.hpp:19-95, datastore.cpp:9-147).
 * Layers are append-only token arrays in HBM; an n-gram occurrence is any (sequence, end) whose last
 * n tokens match, found by a warp-cooperative suffix-match scan (no host index). */
int dbl_store_create(int max_order, int depth, int device, dbl_store_t* out);   /* HierarchicalDatastore(n, d), datastore.hpp:75-79 */
int dbl_store_destroy(dbl_store_t s);
int dbl_store_set_rejected_enabled(dbl_store_t s, int enabled);                  /* rejected_enabled, datastore.hpp:80 */
int dbl_store_set_layer_order(dbl_store_t s, int layer, int max_order);          /* NGramIndex::max_order, datastore.hpp:20 */
int dbl_store_insert(dbl_store_t s, int layer, const int32_t* tokens, int n, int64_t step); /* NGramIndex::insert, datastore.cpp:9-20 */
int dbl_store_record(dbl_store_t s, int layer, const int32_t* tokens, int n);    /* record_accepted / record_rejected, datastore.cpp:134-142 */
int dbl_store_flush_session(dbl_store_t s);                                      /* flush_session, datastore.cpp:144-147 */
int dbl_store_clear_layer(dbl_store_t s, int layer);                             /* NGramIndex::clear, datastore.cpp:28-31 */
int dbl_store_get_step(dbl_store_t s, int64_t* step);                            /* step_counter, datastore.hpp:79 */
int dbl_store_set_step(dbl_store_t s, int64_t step);
/* per-layer sizes; occurrences == NGramIndex::occurrence_count (datastore.cpp:22-26) */
int dbl_store_layer_info(dbl_store_t s, int layer, int64_t* n_seqs, int64_t* n_tokens, int64_t* occurrences);
/* copies back the layer's sequences (dstore-v1 content, datastore.cpp:149-159) */
int dbl_store_layer_read(dbl_store_t s, int layer, int32_t* tokens, int64_t tok_cap, int32_t* seq_lens, int64_t* steps, int64_t seq_cap);
/* HierarchicalDatastore::lookup (datastore.cpp:82-132): one query, host in / host out */
int dbl_store_lookup(dbl_store_t s, const int32_t* ctx, int L, int d, int32_t* cands, int cap,
                     int* n_cands, int* source, int* matched_order);
/* n_q independent queries in ONE launch (one CTA per query); stats accumulate as n_q lookups.
 * q_offsets[n_q+1] index q_tokens; out_cands is n_q x d_cap. */
int dbl_store_lookup_batch(dbl_store_t s, int n_q, const int64_t* q_offsets, const int32_t* q_tokens,
                           const int32_t* depths, int d_cap, int32_t* out_cands, int32_t* out_n,
                           int32_t* out_source, int32_t* out_order);
/* LookupStats (datastore.hpp:39-67): lookups, prior, dynamic, rejected, fallback, misses */
int dbl_store_stats(dbl_store_t s, int64_t out[6]);
/* Device n-gram index over a layer's current sequences: the device form of NGramIndex's n-gram ->
 * occurrence map (datastore.cpp:9-20); build_prior / a dstore-v1 prior build it automatically, later
 * inserts into the layer are scanned until the next build.  Lookup results are identical either way. */
int dbl_store_build_index(dbl_store_t s, int layer);
int dbl_store_index_entries(dbl_store_t s, int layer, int64_t* entries); /* 0: layer not indexed */
/* mean device time of one lookup (iters back-to-back single-CTA lookups on one stream, CUDA events) */
int dbl_store_profile_lookup(dbl_store_t s, const int32_t* ctx, int L, int d, int iters, double* us_per_lookup);

/* ===================================================================== models
 * Replaces specpar::TableModel + forward / forward_batch / argmax_token (model.hpp:18-48,
 * model.cpp:13-81).  Greedy decoding consumes a distribution only through argmax_token (lowest id on
 * ties), so device models return per-row argmax ids; logits/probabilities are available for checks. */
/* TableModel (config 1): n_rows windows of `order` tokens with vocab-wide fp64 rows + fallback row */
int dbl_table_create(int order, int vocab, int64_t n_rows, const int32_t* windows, const double* probs,
                     const double* fallback, int device, dbl_model_t* out);

/* Random-init bf16 decoder-only transformer (Qwen3 / Llama shapes).  No reference counterpart: it
 * stands in for the paper's LLMs behind the same forward_batch contract. */
typedef struct {
    int n_layers, hidden, ffn, n_heads, n_kv_heads, head_dim, vocab;
    int tied_embeddings; /* LM head = embedding matrix */
    int qk_norm;         /* Qwen3 per-head RMSNorm on q and k */
    float rope_theta, rms_eps, init_std;
    int max_seq;         /* KV capacity in tokens */
    uint64_t seed;       /* weights are a pure function of (seed, tensor, index) */
    int tp_rank, tp_size;/* tensor parallel shard (1 = unsharded) */
    float layer_std_scale; /* decoder layers >= scale_from_layer ~ N(0, (init_std * scale)^2); 0 = 1.
                              < 1 gives the labelled "aligned" workload of bench.py: the deep layers only
                              refine the residual stream, so the target's own first layers (early exit,
                              same seed) draft it with alpha > 0 */
    int scale_from_layer;
} dbl_transformer_config;
/* One shard (cfg->tp_rank of cfg->tp_size) or the whole model (tp_size 1) on `device`.  nccl_comm is
 * unused (kept for ABI stability): the tensor-parallel exchange runs inside the forward kernel over
 * peer memory (fwd.cuh), driven by dbl_tp_transformer_create. */
int dbl_transformer_create(const dbl_transformer_config* cfg, int device, void* nccl_comm, dbl_model_t* out);
/* Tensor-parallel target: `world` shards (2..8) of cfg on devices[0..world) — distinct
 * GPUs over NVLink, or repeated devices (shards co-reside) — behind one model handle: forward_batch,
 * run, run_vanilla_ar etc. work unchanged; every shard ends each forward with identical argmax rows. */
int dbl_tp_transformer_create(const dbl_transformer_config* cfg, const int* devices, int world, dbl_model_t* out);
/* One process per GPU: a shard made by dbl_transformer_create (cfg->tp_rank of cfg->tp_size) exports its
 * exchange buffers as 4 CUDA IPC handles (256 bytes into out), the processes all-gather them in rank
 * order (e.g. torch.distributed), and each imports the world x 256 bytes.  From then on every forward of
 * the shard exchanges partial tiles / argmax winners with the other processes inside fwd_kernel, and
 * each process runs the same decode loop (identical decisions on every rank). */
int dbl_tp_ipc_export(dbl_model_t shard, void* out, int64_t cap);
int dbl_tp_ipc_import(dbl_model_t shard, const void* all, int world);
int dbl_model_destroy(dbl_model_t m);
int dbl_model_vocab(dbl_model_t m, int* vocab);
/* bytes of weights streamed per forward on this rank (the roofline numerator's static part) */
int dbl_model_weight_bytes(dbl_model_t m, int64_t* bytes);

/* forward_batch (model.cpp:37-53): |cands|+1 rows, row k = next-token distribution after
 * ctx ⊕ cands[0..k); stateless (transformers recompute the whole context into a scratch KV). */
int dbl_forward_argmax(dbl_model_t m, const int32_t* ctx, int L, const int32_t* cands, int c, int32_t* out_argmax);
/* same rows as fp32 logits (transformer) or fp64 probabilities cast to fp32 (table), (c+1) x vocab */
int dbl_forward_logits(dbl_model_t m, const int32_t* ctx, int L, const int32_t* cands, int c, float* out);
/* the ProbVector rows themselves, fp64 (c+1) x vocab: tables return their rows exactly, transformers
 * softmax(logits) — the same rows the sampled (temperature > 0) decode loop consumes */
int dbl_forward_dists(dbl_model_t m, const int32_t* ctx, int L, const int32_t* cands, int c, double* out);
/* copies a named weight tensor to host (bf16 bits as uint16); for the fp32 torch reference in tests */
int dbl_transformer_get_weight(dbl_model_t m, const char* name, int layer, uint16_t* out, int64_t numel);

/* ===================================================================== decode loop
 * Replaces specpar::run / run_round / compute_metrics / traces_to_jsonl (pipeline.hpp:93-115,
 * pipeline.cpp:15-400) and the harness's run_vanilla_ar (harness.cpp:233-258). */
typedef struct {
    int gamma, depth;
    int draft_retrieval, target_retrieval;
    int concurrent;          /* Engine::Concurrent; the device loop always overlaps draft and target */
    double t_target, t_draft, t_lookup, t_sync; /* LatencyConfig, pipeline.hpp:15-29 */
    int use_graphs;          /* capture the draft chain / target forward in CUDA graphs */
    double temperature;      /* SamplerConfig (model.hpp:11-14): 0 = greedy, > 0 = sampled */
    uint64_t rng_seed;       /* SamplerConfig::rng_seed: per-round streams derive_rng(seed, round, 0/1/2) */
} dbl_pipeline_options;

typedef struct { /* RunMetrics (pipeline.hpp:73-82) + device timing */
    int64_t tokens, rounds;
    double clock, m, amt, speedup, hit_rate;
    int64_t lookups;
    double device_ms;        /* CUDA-event time of the decode loop (prefill excluded) */
    double prefill_ms;       /* CUDA-event time of the prompt prefill */
    double target_fwd_ms;    /* summed CUDA-event time of target verify forwards */
    int64_t target_fwd_count;
    int64_t target_rows;     /* summed verify rows */
    int64_t kernel_launches; /* device kernels launched by the loop (graph nodes counted) */
} dbl_run_metrics;

/* run (pipeline.cpp:264-323).  out: committed tokens after the prompt, truncated to max_new.
 * jsonl: traces_to_jsonl text (may be NULL); jsonl_len receives the full length. */
int dbl_run(dbl_model_t draft, dbl_model_t target, dbl_store_t store, const int32_t* prompt,
            int n_prompt, int max_new, const dbl_pipeline_options* opts, int32_t* out, int cap,
            int* n_out, dbl_run_metrics* metrics, char* jsonl, int64_t jsonl_cap, int64_t* jsonl_len);
/* The decision log of this thread's last dbl_run: the argmax rows the loop consumed, per round
 * n_segs, {matched, emitted[matched+1]} x n_segs, n_spec, rej, correction, ext_matched,
 * ext_emitted[ext_matched+1].  Used to replay the reference's own host loop with the forward
 * excluded (bench.py cpu_baseline / --impl reference).  len receives the full length. */
int dbl_last_run_log(int32_t* buf, int64_t cap, int64_t* len);
/* traces_to_jsonl (pipeline.cpp:373-400) of this thread's last single-sequence run / run_ar /
 * run_serial_sd: also the recovery path when the caller's jsonl buffer was too small (*len = bytes) */
int dbl_last_run_jsonl(char* buf, int64_t cap, int64_t* len);
/* run_vanilla_ar (harness.cpp:233-258), greedy: target-only, one forward per token */
int dbl_run_ar(dbl_model_t target, const int32_t* prompt, int n_prompt, int max_new, double t_target,
               int32_t* out, int cap, int* n_out, dbl_run_metrics* metrics, char* jsonl,
               int64_t jsonl_cap, int64_t* jsonl_len);
/* Sampled decoding (temperature > 0) at wide vocabularies: by default rows of more than 4,096 entries
 * use fixed-order parallel reductions and fp32 tempering (same law, deterministic); with exact
 * sampling on, every row takes the reference's sequential fp64 sums / scan and fp64 pow
 * (model.cpp:55-68, 83-97; verification.cpp:25-58) — decisions bit-identical to the reference at any
 * vocabulary, ~0.5 ms of single-thread fp64 work per 150k-entry row.  Applies to every visible device;
 * set it between runs (a decode in flight on another thread may see either setting). */
int dbl_set_exact_sampling(int on);
/* run_vanilla_ar with a SamplerConfig (harness.cpp:233-258): temperature 0 = dbl_run_ar; > 0 samples
 * each token with Rng(splitmix64(seed ^ 0x6172000000000000)) exactly as the reference */
int dbl_run_ar_sampled(dbl_model_t target, const int32_t* prompt, int n_prompt, int max_new, double t_target,
                       double temperature, uint64_t seed, int32_t* out, int cap, int* n_out,
                       dbl_run_metrics* metrics, char* jsonl, int64_t jsonl_cap, int64_t* jsonl_len);
/* Batched DOUBLE: run() for n_seq (<= 16) independent sequences, one datastore each
 * (stores[b]), sharing every draft-segment and verify forward.  out: n_seq rows of max_new tokens
 * (out_n[b] valid); metrics[b]; jsonl: the sequences' traces_to_jsonl texts back to back, jsonl_lens[b]
 * bytes each (may be NULL).  Each sequence's result equals its own dbl_run. */
int dbl_run_batch(dbl_model_t draft, dbl_model_t target, int n_seq, const dbl_store_t* stores,
                  const int64_t* prompt_off, const int32_t* prompt_tokens, int max_new,
                  const dbl_pipeline_options* opts, int32_t* out, int32_t* out_n, dbl_run_metrics* metrics,
                  char* jsonl, int64_t jsonl_cap, int64_t* jsonl_lens);
/* Batched serving: run_vanilla_ar for n_seq (<= 16) independent prompts in lockstep,
 * ONE forward over all sequences per step (the weight stream is shared).  prompts: prompt_off[n_seq+1]
 * into prompt_tokens.  out: n_seq rows of max_new tokens (row b holds out_n[b] tokens, cut after EOS);
 * every row equals that prompt's own dbl_run_ar output.  device_ms: CUDA-event time of the loop. */
int dbl_run_ar_batch(dbl_model_t target, int n_seq, const int64_t* prompt_off, const int32_t* prompt_tokens,
                     int max_new, int32_t* out, int32_t* out_n, double* device_ms, int64_t* kernel_launches);
/* run_serial_sd (harness.cpp:264-369): draft-then-verify, use_retrieval = draft_retrieval method */
int dbl_run_serial_sd(dbl_model_t draft, dbl_model_t target, dbl_store_t store, const int32_t* prompt,
                      int n_prompt, int max_new, const dbl_pipeline_options* opts, int use_retrieval,
                      int32_t* out, int cap, int* n_out, dbl_run_metrics* metrics, char* jsonl,
                      int64_t jsonl_cap, int64_t* jsonl_len);

/* ===================================================================== verifier + RNG
 * Replaces specpar::Rng / derive_rng (rng.hpp:19-35) and the verifier interface (verification.hpp:
 * 30-53, verification.cpp:19-132).  Probability rows are ragged like the reference's ProbVector:
 * row r = probs[off[r] .. off[r+1]) (fp64), n_rows rows, off[0] = 0.  Draws consume the handle's
 * mt19937_64 stream exactly as the reference consumes its Rng, so outcomes are bit-identical. */
typedef enum { DBL_VERIFY_ALL_ACCEPTED = 0, DBL_VERIFY_CORRECTION = 1, DBL_VERIFY_EXTENSION = 2,
               DBL_VERIFY_RESIDUAL_CORRECTION = 3 } dbl_verify_kind;           /* VerifyKind, verification.hpp:20 */
int dbl_rng_create(uint64_t seed, int device, dbl_rng_t* out);                  /* Rng(seed), rng.hpp:21 */
int dbl_rng_derive(uint64_t seed, uint64_t round, uint64_t lane, int device, dbl_rng_t* out); /* derive_rng, rng.hpp:33-35 */
int dbl_rng_uniform(dbl_rng_t r, double* out, int n);                          /* n x Rng::uniform, rng.hpp:23 */
int dbl_rng_destroy(dbl_rng_t r);
int dbl_accept_prob(const double* p, int np, const double* q, int nq, int32_t x, double* out); /* accept_prob, verification.cpp:19-23 */
int dbl_residual_sample(const double* p, int np, const double* q, int nq, dbl_rng_t r, int32_t* out); /* verification.cpp:40-50 */
int dbl_residual_sample_point_mass(const double* p, int np, int32_t x, dbl_rng_t r, int32_t* out);    /* verification.cpp:52-58 */
/* verify_against_target (verification.cpp:60-78): *first_reject = index or -1 (std::nullopt) */
int dbl_verify_against_target(const int32_t* draft, int n_draft, const double* draft_probs, const int64_t* draft_off,
                              int n_draft_rows, const double* target_probs, const int64_t* target_off,
                              int n_target_rows, double temperature, dbl_rng_t r, int* first_reject);
/* guided_output (verification.cpp:80-132): first_reject = -1 for std::nullopt; committed[cap] */
int dbl_guided_output(const int32_t* draft, int n_draft, const double* draft_probs, const int64_t* draft_off,
                      int n_draft_rows, const int32_t* guide_tokens, int n_guide, const double* guide_probs,
                      const int64_t* guide_off, int n_guide_rows, int first_reject, double temperature, dbl_rng_t r,
                      int32_t* committed, int cap, int* n_committed, int* accepted_len, int* kind);

/* ===================================================================== model-level helpers
 * tempered / argmax_token / sample (model.hpp:40-48, model.cpp:55-97) over explicit fp64 rows.
 * argmax is a block reduction (warp shuffles, ties -> lowest id, RuntimeError when the max <= 0);
 * tempered/sample keep the reference's summation order (single-thread fp64: bit-identical draws). */
int dbl_tempered(const double* dist, int n, double temperature, int device, double* out);    /* model.cpp:55-68 */
int dbl_argmax_token(const double* dist, int n, int device, int32_t* out);                    /* model.cpp:70-81 */
/* argmax_token of n_rows ragged rows (row r = probs[off[r] .. off[r+1])), one CTA per row, one launch */
int dbl_argmax_rows(const double* probs, const int64_t* off, int n_rows, int device, int32_t* out);
int dbl_sample(const double* dist, int n, double temperature, dbl_rng_t r, int device, int32_t* out); /* model.cpp:83-97 */

/* ===================================================================== drafter
 * Replaces accept_with_model / retrieval_forward / iterative_draft / measure_amt (speculation.hpp:34-59,
 * speculation.cpp:7-94).  RetrievalResult: emitted[matched_len + 1] tokens, probs = the model's effective
 * row at every emitted position (greedy: the rows themselves; T > 0: tempered), source. */
typedef struct {
    int matched_len;
    int n_emitted;
    int source;   /* dbl_source (DBL_SRC_MISS when retrieval is off) */
    int n_probs;  /* rows written to probs */
} dbl_retrieval_result;
/* rows: n_dists (= c + 1) ragged fp64 rows; probs (may be NULL) receives rows 0..n_probs of the same
 * lengths, flattened; r may be NULL at temperature 0 (no draw is consumed) */
int dbl_accept_with_model(const double* dists, const int64_t* dist_off, int n_dists, const int32_t* cands, int c,
                          double temperature, dbl_rng_t r, int device, int32_t* emitted, int emitted_cap,
                          double* probs, int64_t probs_cap, dbl_retrieval_result* res);
/* lookup (if use_retrieval) -> one forward_batch of model m over ctx ⊕ candidates -> accept_with_model;
 * probs rows are vocab long.  st may be NULL when use_retrieval is 0. */
int dbl_retrieval_forward(dbl_model_t m, dbl_store_t st, const int32_t* ctx, int L, int depth, double temperature,
                          dbl_rng_t r, int use_retrieval, int32_t* emitted, int emitted_cap, double* probs,
                          int64_t probs_cap, dbl_retrieval_result* res);
/* gamma chained retrieval forwards over the growing context: segs[gamma], tokens = the flattened
 * emissions (DraftChain::tokens), probs (may be NULL) = one vocab row per token */
int dbl_iterative_draft(dbl_model_t m, dbl_store_t st, const int32_t* ctx, int L, int gamma, int depth,
                        double temperature, dbl_rng_t r, int use_retrieval, dbl_retrieval_result* segs,
                        int32_t* tokens, int tokens_cap, int* n_tokens, double* probs, int64_t probs_cap);
int dbl_measure_amt(const int32_t* matched_lens, int n, double* out);                          /* speculation.cpp:88-94 */

/* ===================================================================== decoder state machine
 * PipelineState / RoundTrace / rollback / run_round / compute_metrics / traces_to_jsonl / write_traces
 * (pipeline.hpp:46-115, pipeline.cpp:15-400). */
typedef enum { DBL_MODE_PRE_VERIFY = 0, DBL_MODE_POST_VERIFY = 1, DBL_MODE_AR = 2, DBL_MODE_SERIAL = 3 } dbl_trace_mode;
typedef enum {
    DBL_KIND_PENDING_REJECT = 0, DBL_KIND_EXTEND_KEEP_DRAFT = 1, DBL_KIND_EXTEND_DRAFT_SUBSUMED = 2,
    DBL_KIND_EXTEND_DROP_DRAFT = 3, DBL_KIND_AR_STEP = 4, DBL_KIND_REJECT = 5, DBL_KIND_ALL_ACCEPTED = 6
} dbl_trace_kind;
#define DBL_MAX_SEGS 64
typedef struct { /* RoundTrace (pipeline.hpp:57-71); mode / kind / target_source as enums */
    int64_t round;
    int mode;                          /* dbl_trace_mode */
    int pending, draft_len;
    int n_draft_matched;
    int32_t draft_matched[DBL_MAX_SEGS];
    int target_matched;                /* -1 when target retrieval is off */
    int target_source;                 /* dbl_source */
    int accepted_pending;
    int pending_reject, rejected;
    int committed_count;
    int kind;                          /* dbl_trace_kind */
    double clock_delta;
} dbl_round_trace;
typedef struct { /* PipelineState (pipeline.hpp:46-55) over caller-owned host arrays */
    int32_t* committed;    int64_t n_committed;   int64_t committed_cap;
    int32_t* speculative;  int64_t n_speculative; int64_t speculative_cap;
    int64_t n_spec_probs;  /* |spec_probs| (rows); check_state requires == n_speculative */
    double* spec_probs;    /* T > 0: n_spec_probs x vocab rows, capacity spec_probs_cap rows.  NULL on input =
                              the session's own device rows from its previous round (greedy never reads them) */
    int64_t spec_probs_cap;
    int mode;              /* Mode: 0 PreVerify, 1 PostVerify */
    int prev_tokens;
    int64_t round;
    double clock;          /* SimClock::now */
    int64_t last_committed_len;
} dbl_pipeline_state;
/* rollback (pipeline.cpp:15-30): InvalidArgument beyond the context, LogicError below the boundary */
int dbl_rollback(dbl_pipeline_state* st, int64_t keep_len);
/* run_round needs the draft/target lanes (token buffers + KV) to persist between rounds: a session
 * holds them and re-synchronises them with the state it is given (longest common prefix), so a fresh,
 * rolled-back or copied state runs exactly as the reference's and an unchanged one costs nothing. */
typedef struct dbl_session_s* dbl_session_t;
int dbl_session_create(dbl_model_t draft, dbl_model_t target, dbl_session_t* out);
int dbl_session_destroy(dbl_session_t s);
/* run_round (pipeline.cpp:223-262): one round; st advanced in place.  Capacities are checked before any
 * work: committed_cap >= n_committed + n_speculative + depth + 1, speculative_cap >= gamma * (depth + 1)
 * (and spec_probs_cap rows, when spec_probs is non-NULL at T > 0). */
int dbl_run_round(dbl_session_t s, dbl_store_t store, const dbl_pipeline_options* opts, dbl_pipeline_state* st,
                  dbl_round_trace* trace);
int dbl_compute_metrics(const dbl_round_trace* traces, int n, double t_target, dbl_run_metrics* out); /* pipeline.cpp:325-371 */
int dbl_traces_to_jsonl(const dbl_round_trace* traces, int n, char* buf, int64_t cap, int64_t* len);  /* pipeline.cpp:373-394 */
int dbl_write_traces(const dbl_round_trace* traces, int n, const char* path);                        /* pipeline.cpp:396-400 */
/* RunResult::traces of this thread's last dbl_run / dbl_run_ar(_sampled) / dbl_run_serial_sd */
int dbl_last_run_traces(dbl_round_trace* out, int64_t cap, int64_t* n);
/* HierarchicalDatastore copy (the reference's store is a value type: test_pipeline.cpp:170-187) */
int dbl_store_clone(dbl_store_t src, dbl_store_t* out);
/* build_prior (datastore.cpp:149-159): the store's prior layer := the first `rounds` of n_seqs sequences
 * (seq_off[n_seqs + 1] into tokens), step = index, n-gram order max_order — one bulk upload */
int dbl_build_prior(dbl_store_t s, const int64_t* seq_off, const int32_t* tokens, int n_seqs, int max_order, int rounds);

/* ===================================================================== kernel-level checks
 * Debug entry points used by the parity tests to exercise one kernel against a host reference.
 * dbl_debug_gemm: W [n_out x K] bf16 bits, X [T x K] bf16 bits, padded to tp token columns.
 *   epi 0 StoreBF16 / 4 StoreF32 -> io[T x n_out]; 1 ResidAdd -> io[T x n_out] += W X^T;
 *   2 SiluMul (16 gate | 16 up rows per 32) -> io[T x n_out/2]; 3 Argmax -> argmax[T], io = logits. */
/* Times one model forward of `rows` tokens after a ctx_len context (CUDA events, `iters` repeats):
 * out[8] = forward ms, forward-kernel ms (per-launch events), algorithmic bytes (SURVEY §8(d):
 * weights + KV + embedding rows), timed launches, kernel launches (per forward), token columns,
 * last timed launch ms, its bytes.  Feeds bench.py's roofline. */
int dbl_profile_forward(dbl_model_t m, int ctx_len, int rows, int iters, double* out);
/* DBL_GEMM_TRACE=1 timeline of the GEMM launches since the last call: stamps[n][320][4] (%globaltimer
 * ns per CTA: resident, dependency resolved, last load issued, epilogue done), grid and weight bytes */
int dbl_debug_gemm_trace(uint64_t* stamps, int64_t cap, int32_t* grids, int64_t* bytes, int* n_launches);
/* DBL_FWD_TRACE=1: per-(phase, CTA) stamps of the most recent stream forward, [n_ph][grid][16] */
int dbl_debug_fwd_trace(uint64_t* stamps, int64_t cap, int* n_ph, int* grid);
/* back-to-back launches of one GEMM shape, ms per launch (weights rotate over `chain` copies) */
int dbl_debug_gemm_bench(int epi, int n_out, int K, int tp, int iters, int chain, double* ms_per_launch);
int dbl_debug_gemm(int epi, const uint16_t* W, int n_out, int K, const uint16_t* X, int T, int tp,
                   int n_valid, float* io, int32_t* argmax);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* DOUBLE_B200_H */
