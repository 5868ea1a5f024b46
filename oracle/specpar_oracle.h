/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the DOUBLE decode loop.
 *
 * A plain-C restatement of the reference's greedy decode path (/root/reference/proj/src), used by
 * tests/ as the checker and by bench.py's cpu_baseline leg.  The product (libdouble_b200.so) never
 * links, loads or calls it.  Every function cites the reference file:line it restates.
 *
 * Parity of this restatement is PINNED against the reference itself: tests/golden/ holds vectors
 * produced by the unmodified reference (oracle/_ref, built from /root/reference by oracle/Makefile)
 * and tests/test_oracle.py checks this file against them (config-1 traces and model/prior
 * serialisations by sha256, the 100-config acceptance set, lookup known-answer cases).
 *
 * The decode loop is greedy (temperature 0): there the reference consumes a distribution solely
 * through argmax_token (model.cpp:70-81), so models enter the loop as "argmax row" callbacks.  The
 * verifier functions (verification.cpp:19-132) are restated for T >= 0 over explicit rows.
 */
#ifndef SPECPAR_ORACLE_H
#define SPECPAR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:8-35 ---- */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
uint64_t orc_splitmix64(uint64_t x);
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
double orc_uniform(orc_mt64* g);

/* ---- harness.cpp:151-186 ---- corpus flattened into tokens[length]; seq_lens[n_seqs] */
int orc_gen_corpus(int vocab, double rho, int length, uint64_t seed, int* tokens, int* seq_lens,
                   int* n_seqs);

/* ---- model.cpp:13-26, 70-81, 99-152, 174-228 ---- */
typedef struct orc_table orc_table;
orc_table* orc_table_build(const int* tokens, const int* seq_lens, int n_seqs, int order,
                           double smoothing, int vocab);
orc_table* orc_table_parse(const char* model_v1_text);
void orc_table_free(orc_table* t);
int orc_table_vocab(const orc_table* t);
int orc_table_order(const orc_table* t);
/* model-v1 text (malloc'd, caller frees with orc_free) */
char* orc_table_serialize(const orc_table* t);
/* distribution after ctx[0..L) ; returns pointer into the table (row or fallback) */
const double* orc_table_row(const orc_table* t, const int* ctx, int L);
/* argmax with lowest-id tie-break; -1 on a degenerate row (max <= 0) */
int orc_argmax(const double* p, int n);
/* callback-compatible batch argmax: rows for ctx, ctx+cands[0..1), ... (c+1 rows) */
int orc_table_argmax_rows(void* table, const int* ctx, int L, const int* cands, int c, int* out);

/* ---- datastore.cpp:9-147 ---- */
enum { ORC_PRIOR = 0, ORC_DYNAMIC = 1, ORC_REJECTED = 2, ORC_CONTEXT = 3, ORC_MISS = 4 };
typedef struct orc_store orc_store;
orc_store* orc_store_new(int max_order, int depth);
void orc_store_free(orc_store* s);
void orc_store_set_rejected_enabled(orc_store* s, int on);
int orc_layer_insert(orc_store* s, int layer, const int* toks, int n, long step);
long orc_layer_occurrences(const orc_store* s, int layer);
int orc_layer_num_seqs(const orc_store* s, int layer);
int orc_store_record(orc_store* s, int layer, const int* toks, int n);
void orc_store_flush(orc_store* s);
long orc_store_step(const orc_store* s);
int orc_store_lookup(orc_store* s, const int* ctx, int L, int d, int* out_cands, int* n_out,
                     int* source, int* order);
void orc_store_stats(const orc_store* s, long* out6);
/* dstore-v1 (datastore.cpp:161-205) : loads sequences into `layer` with steps 0..n-1 */
int orc_store_load_dstore(orc_store* s, int layer, const char* text);
char* orc_store_serialize_layer(const orc_store* s, int layer);

/* ---- pipeline.cpp:15-400, speculation.cpp:7-86, verification.cpp:60-78 ---- */
typedef int (*orc_argmax_fn)(void* user, const int* ctx, int L, const int* cands, int c, int* out);
typedef struct {
    int gamma, depth, draft_retrieval, target_retrieval;
    double t_target, t_draft, t_lookup, t_sync;
} orc_opts;
/* metrics[8] = tokens, rounds, clock, m, amt, speedup, hit_rate, lookups (pipeline.hpp:73-82) */
int orc_run(int draft_vocab, orc_argmax_fn dfn, void* duser, int target_vocab, orc_argmax_fn tfn,
            void* tuser, orc_store* store, const int* prompt, int n_prompt, int max_new,
            const orc_opts* opts, int* out_tokens, int cap, int* n_out, char** jsonl,
            double* metrics);
/* run_vanilla_ar (harness.cpp:233-258), greedy */
int orc_run_ar(int target_vocab, orc_argmax_fn tfn, void* tuser, const int* prompt, int n_prompt,
               int max_new, double t_target, int* out_tokens, int cap, int* n_out, char** jsonl,
               double* metrics);
/* run_method_on(parse_config(text), build_setup, method) (harness.cpp:55-122, 188-210, 403-429) */
int orc_run_config(const char* cfg_text, const char* method, int* out_tokens, int cap, int* n_out,
                   char** jsonl, double* metrics);

/* Replay models: serve the argmax rows a device run consumed (its decision log, dbl_last_run_log)
 * so the reference/oracle host loop can be timed on the same workload with the forward excluded. */
typedef struct orc_replay orc_replay;
orc_replay* orc_replay_new(const int* log, long len);
void orc_replay_free(orc_replay* r);
void orc_replay_reset(orc_replay* r);
int orc_replay_draft(void* replay, const int* ctx, int L, const int* cands, int c, int* out);
int orc_replay_target(void* replay, const int* ctx, int L, const int* cands, int c, int* out);

/* ---- verification.cpp:19-132 (T >= 0): ragged rows row r = probs[off[r] .. off[r+1]);
 *      returns 0, -1 (std::invalid_argument) or -2 (std::runtime_error) ---- */
int orc_accept_prob(const double* p, int np, const double* q, int nq, int x, double* out);
int orc_residual_sample(const double* p, int np, const double* q, int nq, orc_mt64* g, int* out);
int orc_residual_point_mass(const double* p, int np, int x, orc_mt64* g, int* out);
int orc_verify_against_target(const int* draft, int n_draft, const double* dp, const int64_t* doff, int n_dp,
                              const double* tp, const int64_t* toff, int n_tp, double temperature, orc_mt64* g,
                              int* first_reject);
int orc_guided_output(const int* draft, int n_draft, const double* dp, const int64_t* doff, int n_dp,
                      const int* gtok, int n_gtok, const double* gp, const int64_t* goff, int n_gp,
                      int first_reject, double temperature, orc_mt64* g, int* committed, int cap,
                      int* n_committed, int* accepted_len, int* kind);

const char* orc_last_error(void);
void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
