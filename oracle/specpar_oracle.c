/* TEST INFRASTRUCTURE ONLY — CPU oracle (restatement) of the reference DOUBLE decode loop.
 * See specpar_oracle.h for scope.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this file's library; the product never does.
 *
 * Parity: pinned against the unmodified reference via tests/golden/ (see tests/test_oracle.py).
 */
#define _GNU_SOURCE
#include "specpar_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}
const char* orc_last_error(void) { return g_err; }
void orc_free(void* p) { free(p); }

/* ------------------------------------------------------------------ small growable buffers */
typedef struct { int* v; long n, cap; } ivec;
static void iv_reserve(ivec* a, long want) {
    if (want <= a->cap) return;
    long c = a->cap ? a->cap : 16;
    while (c < want) c *= 2;
    a->v = (int*)realloc(a->v, (size_t)c * sizeof(int));
    a->cap = c;
}
static void iv_push(ivec* a, int x) { iv_reserve(a, a->n + 1); a->v[a->n++] = x; }
static void iv_append(ivec* a, const int* x, long n) {
    if (n <= 0) return;
    iv_reserve(a, a->n + n);
    memcpy(a->v + a->n, x, (size_t)n * sizeof(int));
    a->n += n;
}
static void iv_free(ivec* a) { free(a->v); a->v = NULL; a->n = a->cap = 0; }

typedef struct { char* s; long n, cap; } sbuf;
static void sb_put(sbuf* b, const char* s) {
    long k = (long)strlen(s);
    if (b->n + k + 1 > b->cap) {
        long c = b->cap ? b->cap : 256;
        while (c < b->n + k + 1) c *= 2;
        b->s = (char*)realloc(b->s, (size_t)c);
        b->cap = c;
    }
    memcpy(b->s + b->n, s, (size_t)k + 1);
    b->n += k;
}
static void sb_int(sbuf* b, long x) { char t[32]; snprintf(t, sizeof t, "%ld", x); sb_put(b, t); }

/* ------------------------------------------------------------------ rng.hpp:8-35 */
uint64_t orc_splitmix64(uint64_t x) { /* rng.hpp:8-13 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d49bb133111ebULL;
    return x ^ (x >> 31);
}
/* std::mt19937_64 (the engine behind specpar::Rng, rng.hpp:19-30), standard parameters */
void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
double orc_uniform(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; } /* rng.hpp:24 */

/* ------------------------------------------------------------------ harness.cpp:151-186 */
int orc_gen_corpus(int vocab, double rho, int length, uint64_t seed, int* tokens, int* seq_lens,
                   int* n_seqs) {
    if (vocab < 4) return fail("vocab must be >= 4");
    if (rho < 0.0 || rho > 1.0) return fail("rho out of [0,1]");
    if (length < 1) return fail("length must be >= 1");
    orc_mt64 g;
    orc_mt64_seed(&g, orc_splitmix64(seed ^ 0x636f727075730000ULL));
    const int lo = 1, hi = vocab - 2;
    ivec st = {0};
    while (st.n < length) {
        const int replay = st.n >= 4 && orc_uniform(&g) < rho; /* short-circuit as in C++ */
        if (replay) {
            const long span = 4 + (long)(orc_uniform(&g) * 13.0);
            const long start = (long)(orc_uniform(&g) * (double)st.n);
            const long end = start + span < st.n ? start + span : st.n;
            for (long i = start; i < end; ++i) iv_push(&st, st.v[i]);
        } else {
            const int span = 1 + (int)(orc_uniform(&g) * 4.0);
            for (int i = 0; i < span; ++i)
                iv_push(&st, lo + (int)(orc_uniform(&g) * (double)(hi - lo + 1)));
        }
    }
    memcpy(tokens, st.v, (size_t)length * sizeof(int));
    int k = 0;
    for (int at = 0; at < length; at += 64) seq_lens[k++] = (length - at) < 64 ? (length - at) : 64;
    *n_seqs = k;
    iv_free(&st);
    return 0;
}

/* ------------------------------------------------------------------ model.cpp */
struct orc_table {
    int order, vocab;
    double smoothing;
    long n_rows, cap;       /* open-addressing hash: window -> row index */
    int* windows;           /* n_rows * order */
    double* probs;          /* n_rows * vocab */
    long* slots;            /* cap entries, -1 empty */
    double* fallback;       /* vocab */
};

static uint64_t hash_window(const int* w, int order) {
    uint64_t h = 1469598103934665603ULL;
    for (int i = 0; i < order; ++i) h = (h ^ (uint32_t)w[i]) * 1099511628211ULL;
    return orc_splitmix64(h);
}
static long table_find(const orc_table* t, const int* w) {
    if (!t->cap) return -1;
    uint64_t h = hash_window(w, t->order) & (uint64_t)(t->cap - 1);
    for (;;) {
        long r = t->slots[h];
        if (r < 0) return -1;
        if (!memcmp(t->windows + r * t->order, w, (size_t)t->order * sizeof(int))) return r;
        h = (h + 1) & (uint64_t)(t->cap - 1);
    }
}
static void table_rehash(orc_table* t, long cap) {
    free(t->slots);
    t->cap = cap;
    t->slots = (long*)malloc((size_t)cap * sizeof(long));
    for (long i = 0; i < cap; ++i) t->slots[i] = -1;
    for (long r = 0; r < t->n_rows; ++r) {
        uint64_t h = hash_window(t->windows + r * t->order, t->order) & (uint64_t)(cap - 1);
        while (t->slots[h] >= 0) h = (h + 1) & (uint64_t)(cap - 1);
        t->slots[h] = r;
    }
}
/* returns row index, creating a zero row if absent */
static long table_get_or_add(orc_table* t, const int* w, long* rows_cap) {
    long r = table_find(t, w);
    if (r >= 0) return r;
    if (t->n_rows + 1 > *rows_cap) {
        *rows_cap = *rows_cap ? *rows_cap * 2 : 64;
        t->windows = (int*)realloc(t->windows, (size_t)(*rows_cap * t->order) * sizeof(int));
        t->probs = (double*)realloc(t->probs, (size_t)(*rows_cap * t->vocab) * sizeof(double));
    }
    r = t->n_rows++;
    memcpy(t->windows + r * t->order, w, (size_t)t->order * sizeof(int));
    memset(t->probs + r * t->vocab, 0, (size_t)t->vocab * sizeof(double));
    if (t->n_rows * 2 > t->cap) table_rehash(t, t->cap ? t->cap * 2 : 64);
    else {
        uint64_t h = hash_window(w, t->order) & (uint64_t)(t->cap - 1);
        while (t->slots[h] >= 0) h = (h + 1) & (uint64_t)(t->cap - 1);
        t->slots[h] = r;
    }
    return r;
}

/* window_of, model.cpp:13-21: last `order` tokens, left-padded with BOS (0) */
static void window_of(int order, const int* ctx, long n, int* w) {
    const long take = n < order ? n : order;
    for (int i = 0; i < order; ++i) w[i] = 0;
    for (long i = 0; i < take; ++i) w[order - take + i] = ctx[n - take + i];
}

orc_table* orc_table_build(const int* tokens, const int* seq_lens, int n_seqs, int order,
                           double smoothing, int vocab) { /* model.cpp:99-152 */
    if (n_seqs <= 0) { fail("empty corpus"); return NULL; }
    if (order < 1) { fail("order must be >= 1"); return NULL; }
    if (smoothing < 0.0) { fail("smoothing must be >= 0"); return NULL; }
    orc_table* t = (orc_table*)calloc(1, sizeof *t);
    t->order = order; t->vocab = vocab; t->smoothing = smoothing;
    long rows_cap = 0;
    double* global = (double*)calloc((size_t)vocab, sizeof(double));
    int* w = (int*)malloc((size_t)order * sizeof(int));
    long at = 0;
    for (int s = 0; s < n_seqs; ++s) {
        const int* seq = tokens + at;
        const long len = seq_lens[s];
        for (long i = 0; i < len; ++i) {
            if (seq[i] < 0 || seq[i] >= vocab) {
                fail("corpus token out of range");
                free(global); free(w); orc_table_free(t);
                return NULL;
            }
            global[seq[i]] += 1.0;
            if (i + 1 < len) {
                const long lo = i + 1 >= order ? i + 1 - order : 0;
                window_of(order, seq + lo, i + 1 - lo, w);
                long r = table_get_or_add(t, w, &rows_cap);
                t->probs[r * vocab + seq[i + 1]] += 1.0;
            }
        }
        at += len;
    }
    for (long r = 0; r < t->n_rows; ++r) { /* normalize, model.cpp:127-137 */
        double* p = t->probs + r * vocab;
        double sum = 0.0;
        for (int k = 0; k < vocab; ++k) { p[k] = p[k] + smoothing; sum += p[k]; }
        for (int k = 0; k < vocab; ++k) p[k] /= sum;
    }
    double gsum = 0.0; /* fallback, model.cpp:141-150 */
    for (int k = 0; k < vocab; ++k) gsum += global[k];
    const double sm = smoothing > 1e-12 ? smoothing : 1e-12;
    t->fallback = (double*)malloc((size_t)vocab * sizeof(double));
    for (int k = 0; k < vocab; ++k) t->fallback[k] = (global[k] + sm) / (gsum + sm * vocab);
    free(global); free(w);
    return t;
}

void orc_table_free(orc_table* t) {
    if (!t) return;
    free(t->windows); free(t->probs); free(t->slots); free(t->fallback); free(t);
}
int orc_table_vocab(const orc_table* t) { return t->vocab; }
int orc_table_order(const orc_table* t) { return t->order; }

const double* orc_table_row(const orc_table* t, const int* ctx, int L) { /* model.cpp:23-26 */
    int w[64];
    window_of(t->order, ctx, L, w);
    long r = table_find(t, w);
    return r < 0 ? t->fallback : t->probs + r * t->vocab;
}

int orc_argmax(const double* p, int n) { /* model.cpp:70-81: strict '>' keeps the lowest id */
    int best = 0;
    double bp = -1.0;
    for (int i = 0; i < n; ++i)
        if (p[i] > bp) { bp = p[i]; best = i; }
    return bp <= 0.0 ? -1 : best;
}

int orc_table_argmax_rows(void* table, const int* ctx, int L, const int* cands, int c, int* out) {
    const orc_table* t = (const orc_table*)table; /* forward_batch, model.cpp:37-53 */
    if (L <= 0) return fail("forward_batch: empty context");
    if (t->order > 64) return fail("order too large for the oracle");
    int* buf = (int*)malloc((size_t)(L + c) * sizeof(int));
    memcpy(buf, ctx, (size_t)L * sizeof(int));
    if (c) memcpy(buf + L, cands, (size_t)c * sizeof(int));
    int rc = 0;
    for (int k = 0; k <= c; ++k) {
        out[k] = orc_argmax(orc_table_row(t, buf, L + k), t->vocab);
        if (out[k] < 0) { rc = fail("degenerate distribution"); break; }
    }
    free(buf);
    return rc;
}

static int cmp_order;
static const int* cmp_windows;
static int cmp_rows(const void* a, const void* b) { /* std::map<TokenSeq> order: lexicographic */
    const int* x = cmp_windows + (long)(*(const long*)a) * cmp_order;
    const int* y = cmp_windows + (long)(*(const long*)b) * cmp_order;
    for (int i = 0; i < cmp_order; ++i)
        if (x[i] != y[i]) return x[i] < y[i] ? -1 : 1;
    return 0;
}
static void put_probs(sbuf* b, const double* p, int n) {
    char t[64];
    for (int i = 0; i < n; ++i) { snprintf(t, sizeof t, " %.17g", p[i]); sb_put(b, t); }
}
char* orc_table_serialize(const orc_table* t) { /* model-v1, model.cpp:174-197 */
    sbuf b = {0};
    char t0[128];
    snprintf(t0, sizeof t0, "model-v1 %d %d %.17g\n", t->vocab, t->order, t->smoothing);
    sb_put(&b, t0);
    long* idx = (long*)malloc((size_t)(t->n_rows ? t->n_rows : 1) * sizeof(long));
    for (long r = 0; r < t->n_rows; ++r) idx[r] = r;
    cmp_order = t->order; cmp_windows = t->windows;
    qsort(idx, (size_t)t->n_rows, sizeof(long), cmp_rows);
    for (long i = 0; i < t->n_rows; ++i) {
        const int* w = t->windows + idx[i] * t->order;
        for (int k = 0; k < t->order; ++k) {
            if (k) sb_put(&b, " ");
            sb_int(&b, w[k]);
        }
        sb_put(&b, " :");
        put_probs(&b, t->probs + idx[i] * t->vocab, t->vocab);
        sb_put(&b, "\n");
    }
    sb_put(&b, "fallback :");
    put_probs(&b, t->fallback, t->vocab);
    sb_put(&b, "\n");
    free(idx);
    return b.s;
}

orc_table* orc_table_parse(const char* text) { /* model.cpp:199-228 */
    orc_table* t = (orc_table*)calloc(1, sizeof *t);
    char magic[32] = {0};
    int consumed = 0;
    if (sscanf(text, "%31s %d %d %lf%n", magic, &t->vocab, &t->order, &t->smoothing, &consumed) < 4 ||
        strcmp(magic, "model-v1") || t->order < 1 || t->order > 64 || t->vocab < 1) {
        fail("model-v1: bad header");
        free(t);
        return NULL;
    }
    long rows_cap = 0;
    const char* p = strchr(text, '\n');
    int w[64];
    while (p && *p) {
        ++p;
        while (*p == ' ') ++p;
        if (*p == '\n' || *p == 0) continue;
        double* row;
        if (!strncmp(p, "fallback", 8)) {
            p = strchr(p, ':') + 1;
            t->fallback = (double*)malloc((size_t)t->vocab * sizeof(double));
            row = t->fallback;
        } else {
            for (int k = 0; k < t->order; ++k) w[k] = (int)strtol(p, (char**)&p, 10);
            while (*p == ' ') ++p;
            if (*p != ':') { fail("model-v1: window length mismatch"); orc_table_free(t); return NULL; }
            ++p;
            const long r = table_get_or_add(t, w, &rows_cap); /* may realloc probs */
            row = t->probs + r * t->vocab;
        }
        for (int k = 0; k < t->vocab; ++k) {
            char* e;
            row[k] = strtod(p, &e);
            if (e == p) { fail("model-v1: truncated probability row"); orc_table_free(t); return NULL; }
            p = e;
        }
        p = strchr(p, '\n');
    }
    if (!t->fallback) { fail("model-v1: missing fallback row"); orc_table_free(t); return NULL; }
    return t;
}

/* ------------------------------------------------------------------ datastore.cpp */
typedef struct {
    int max_order;
    ivec tokens;     /* all sequences back to back */
    ivec starts, lens;
    long* steps; long steps_cap;
} layer_t;

struct orc_store {
    layer_t layer[3];
    int max_order, depth, rejected_enabled;
    long step_counter;
    long stats[6]; /* lookups, prior, dynamic, rejected, fallback, misses (datastore.hpp:39-67) */
};

orc_store* orc_store_new(int max_order, int depth) { /* datastore.hpp:75-79 */
    orc_store* s = (orc_store*)calloc(1, sizeof *s);
    s->max_order = max_order;
    s->depth = depth;
    s->rejected_enabled = 1;
    for (int l = 0; l < 3; ++l) s->layer[l].max_order = max_order;
    return s;
}
static void layer_clear(layer_t* L) { /* NGramIndex::clear, datastore.cpp:28-31 */
    L->tokens.n = L->starts.n = L->lens.n = 0;
}
void orc_store_free(orc_store* s) {
    if (!s) return;
    for (int l = 0; l < 3; ++l) {
        iv_free(&s->layer[l].tokens); iv_free(&s->layer[l].starts); iv_free(&s->layer[l].lens);
        free(s->layer[l].steps);
    }
    free(s);
}
void orc_store_set_rejected_enabled(orc_store* s, int on) { s->rejected_enabled = on; }

int orc_layer_insert(orc_store* s, int layer, const int* toks, int n, long step) {
    /* NGramIndex::insert, datastore.cpp:9-20.  The occurrence lists are implicit: an occurrence of
     * an n-gram is any (seq, end) whose last n tokens equal it, which is what insert() enumerates. */
    if (layer < 0 || layer > 2) return fail("bad layer");
    if (n <= 0) return fail("insert: empty token sequence");
    layer_t* L = &s->layer[layer];
    if (L->lens.n + 1 > L->steps_cap) {
        L->steps_cap = L->steps_cap ? L->steps_cap * 2 : 16;
        L->steps = (long*)realloc(L->steps, (size_t)L->steps_cap * sizeof(long));
    }
    L->steps[L->lens.n] = step;
    iv_push(&L->starts, (int)L->tokens.n);
    iv_push(&L->lens, n);
    iv_append(&L->tokens, toks, n);
    return 0;
}
long orc_layer_occurrences(const orc_store* s, int layer) { /* occurrence_count, datastore.cpp:22-26 */
    const layer_t* L = &s->layer[layer];
    long total = 0;
    for (long i = 0; i < L->lens.n; ++i)
        for (int k = 1; k <= L->max_order; ++k)
            if (L->lens.v[i] >= k) total += L->lens.v[i] - k + 1;
    return total;
}
int orc_layer_num_seqs(const orc_store* s, int layer) { return (int)s->layer[layer].lens.n; }
long orc_store_step(const orc_store* s) { return s->step_counter; }

int orc_store_record(orc_store* s, int layer, const int* toks, int n) { /* datastore.cpp:134-142 */
    if (n <= 0) return 0;
    return orc_layer_insert(s, layer, toks, n, s->step_counter++);
}
void orc_store_flush(orc_store* s) { /* datastore.cpp:144-147 (step_counter is kept) */
    layer_clear(&s->layer[ORC_DYNAMIC]);
    layer_clear(&s->layer[ORC_REJECTED]);
}
void orc_store_stats(const orc_store* s, long* out6) { memcpy(out6, s->stats, sizeof s->stats); }

/* best_occurrence, datastore.cpp:49-71: lexicographic max of (step, avail, seq_id, end_pos) over
 * occurrences with avail = min(remaining, d) > 0.  Returns 1 and (seq, end) when found. */
static int best_occurrence(const layer_t* L, const int* key, int n, int d, long* bseq, long* bend) {
    if (n > L->max_order) return 0;
    int found = 0;
    long b_step = 0, b_avail = 0, b_seq = 0, b_end = 0;
    for (long q = 0; q < L->lens.n; ++q) {
        const int* seq = L->tokens.v + L->starts.v[q];
        const long len = L->lens.v[q];
        for (long end = n - 1; end < len; ++end) {
            int match = 1;
            for (int j = 0; j < n; ++j)
                if (seq[end - n + 1 + j] != key[j]) { match = 0; break; }
            if (!match) continue;
            const long remaining = len - end - 1;
            const long avail = remaining < d ? remaining : d;
            if (avail <= 0) continue;
            const long step = L->steps[q];
            if (!found || step > b_step ||
                (step == b_step &&
                 (avail > b_avail ||
                  (avail == b_avail && (q > b_seq || (q == b_seq && end > b_end)))))) {
                found = 1; b_step = step; b_avail = avail; b_seq = q; b_end = end;
            }
        }
    }
    *bseq = b_seq; *bend = b_end;
    return found;
}

int orc_store_lookup(orc_store* s, const int* ctx, int L, int d, int* out_cands, int* n_out,
                     int* source, int* order) { /* HierarchicalDatastore::lookup, datastore.cpp:82-132 */
    if (L <= 0) return fail("lookup: empty context");
    s->stats[0]++;
    const int nmax = s->max_order < L ? s->max_order : L;
    for (int n = nmax; n >= 1; --n) {
        const int* key = ctx + L - n;
        for (int l = 0; l < 3; ++l) {
            if (l == ORC_REJECTED && !s->rejected_enabled) continue;
            long q, end;
            if (best_occurrence(&s->layer[l], key, n, d, &q, &end)) {
                const layer_t* Ly = &s->layer[l];
                const int* seq = Ly->tokens.v + Ly->starts.v[q];
                const long from = end + 1;
                const long to = from + d < Ly->lens.v[q] ? from + d : Ly->lens.v[q]; /* :73-78 */
                for (long i = from; i < to; ++i) out_cands[i - from] = seq[i];
                *n_out = (int)(to - from);
                *source = l;
                *order = n;
                s->stats[1 + l]++;
                return 0;
            }
        }
    }
    const int nf = s->max_order < L - 1 ? s->max_order : L - 1; /* PLD fallback, :109-128 */
    for (int n = nf; n >= 1; --n) {
        for (int end = L - 2; end >= n - 1; --end) {
            int match = 1;
            for (int j = 0; j < n; ++j)
                if (ctx[end - j] != ctx[L - 1 - j]) { match = 0; break; }
            if (match) {
                s->stats[4]++;
                const int from = end + 1;
                const int to = from + d < L ? from + d : L;
                for (int i = from; i < to; ++i) out_cands[i - from] = ctx[i];
                *n_out = to > from ? to - from : 0;
                *source = ORC_CONTEXT;
                *order = n;
                return 0;
            }
        }
    }
    s->stats[5]++;
    *n_out = 0;
    *source = ORC_MISS;
    *order = 0;
    return 0;
}

int orc_store_load_dstore(orc_store* s, int layer, const char* text) { /* parse_index, :161-187 */
    char magic[32] = {0};
    int mo = 0;
    long count = 0;
    if (sscanf(text, "%31s %d %ld", magic, &mo, &count) < 3 || strcmp(magic, "dstore-v1"))
        return fail("dstore-v1: bad header");
    layer_clear(&s->layer[layer]);
    s->layer[layer].max_order = mo;
    const char* p = strchr(text, '\n');
    ivec seq = {0};
    for (long i = 0; i < count; ++i) {
        if (!p || !*p) { iv_free(&seq); return fail("dstore-v1: truncated"); }
        ++p;
        const char* eol = strchr(p, '\n');
        if (!eol) eol = p + strlen(p);
        seq.n = 0;
        while (p < eol) {
            char* e;
            long v = strtol(p, &e, 10);
            if (e == p) break;
            iv_push(&seq, (int)v);
            p = e;
        }
        p = eol;
        if (orc_layer_insert(s, layer, seq.v, (int)seq.n, i)) { iv_free(&seq); return -1; }
    }
    iv_free(&seq);
    return 0;
}

char* orc_store_serialize_layer(const orc_store* s, int layer) { /* serialize_index, :149-159 */
    const layer_t* L = &s->layer[layer];
    sbuf b = {0};
    char t[96];
    snprintf(t, sizeof t, "dstore-v1 %d %ld\n", L->max_order, L->lens.n);
    sb_put(&b, t);
    for (long q = 0; q < L->lens.n; ++q) {
        for (int i = 0; i < L->lens.v[q]; ++i) {
            if (i) sb_put(&b, " ");
            sb_int(&b, L->tokens.v[L->starts.v[q] + i]);
        }
        sb_put(&b, "\n");
    }
    return b.s;
}

/* ------------------------------------------------------------------ traces (pipeline.hpp:57-71) */
typedef struct {
    long round;
    const char* mode;
    int pending, draft_len;
    ivec draft_matched;
    int target_matched;
    const char* target_source;
    int accepted_pending, pending_reject, rejected, committed_count;
    const char* kind;
    double clock_delta;
} trace_t;
typedef struct { trace_t* v; long n, cap; } tvec;
static trace_t* tv_new(tvec* a) {
    if (a->n + 1 > a->cap) {
        a->cap = a->cap ? a->cap * 2 : 64;
        a->v = (trace_t*)realloc(a->v, (size_t)a->cap * sizeof(trace_t));
    }
    trace_t* t = &a->v[a->n++];
    memset(t, 0, sizeof *t);
    t->mode = ""; t->target_source = ""; t->kind = ""; t->target_matched = -1;
    return t;
}
static void tv_free(tvec* a) {
    for (long i = 0; i < a->n; ++i) iv_free(&a->v[i].draft_matched);
    free(a->v);
}

/* nlohmann::json number formatting: shortest round-trip digits, then format_buffer with
 * min_exp = -4, max_exp = 15 ("1.0", "2.5", "0.001", "1e-05", "1e+16") */
static void json_double(sbuf* b, double x) {
    char digits[40], tmp[64];
    if (x == 0.0) { sb_put(b, signbit(x) ? "-0.0" : "0.0"); return; }
    int prec = 1;
    for (; prec <= 17; ++prec) {
        snprintf(tmp, sizeof tmp, "%.*e", prec - 1, x);
        if (strtod(tmp, NULL) == x) break;
    }
    char* p = tmp;
    int neg = 0;
    if (*p == '-') { neg = 1; ++p; }
    int k = 0;
    for (; *p && *p != 'e'; ++p) if (*p != '.') digits[k++] = *p;
    digits[k] = 0;
    int e10 = atoi(p + 1);
    while (k > 1 && digits[k - 1] == '0') digits[--k] = 0;
    const int n = e10 + 1; /* decimal point position */
    char out[80];
    int o = 0;
    if (neg) out[o++] = '-';
    if (k <= n && n <= 15) {
        memcpy(out + o, digits, (size_t)k); o += k;
        for (int i = k; i < n; ++i) out[o++] = '0';
        out[o++] = '.'; out[o++] = '0';
    } else if (0 < n && n <= 15) {
        memcpy(out + o, digits, (size_t)n); o += n;
        out[o++] = '.';
        memcpy(out + o, digits + n, (size_t)(k - n)); o += k - n;
    } else if (-4 < n && n <= 0) {
        out[o++] = '0'; out[o++] = '.';
        for (int i = 0; i < -n; ++i) out[o++] = '0';
        memcpy(out + o, digits, (size_t)k); o += k;
    } else {
        out[o++] = digits[0];
        if (k > 1) { out[o++] = '.'; memcpy(out + o, digits + 1, (size_t)(k - 1)); o += k - 1; }
        const int e = n - 1;
        o += snprintf(out + o, sizeof out - (size_t)o, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    }
    out[o] = 0;
    sb_put(b, out);
}

static char* traces_jsonl(const tvec* tr) { /* traces_to_jsonl, pipeline.cpp:373-394 */
    sbuf b = {0};
    sb_put(&b, "");
    for (long i = 0; i < tr->n; ++i) {
        const trace_t* t = &tr->v[i];
        sb_put(&b, "{\"round\":"); sb_int(&b, t->round);
        sb_put(&b, ",\"mode\":\""); sb_put(&b, t->mode);
        sb_put(&b, "\",\"pending\":"); sb_int(&b, t->pending);
        sb_put(&b, ",\"draft_len\":"); sb_int(&b, t->draft_len);
        sb_put(&b, ",\"draft_matched\":[");
        for (long k = 0; k < t->draft_matched.n; ++k) {
            if (k) sb_put(&b, ",");
            sb_int(&b, t->draft_matched.v[k]);
        }
        sb_put(&b, "],\"target_matched\":"); sb_int(&b, t->target_matched);
        sb_put(&b, ",\"target_source\":\""); sb_put(&b, t->target_source);
        sb_put(&b, "\",\"accepted_pending\":"); sb_int(&b, t->accepted_pending);
        sb_put(&b, ",\"pending_reject\":"); sb_put(&b, t->pending_reject ? "true" : "false");
        sb_put(&b, ",\"rejected\":"); sb_put(&b, t->rejected ? "true" : "false");
        sb_put(&b, ",\"committed\":"); sb_int(&b, t->committed_count);
        sb_put(&b, ",\"kind\":\""); sb_put(&b, t->kind);
        sb_put(&b, "\",\"clock_delta\":"); json_double(&b, t->clock_delta);
        sb_put(&b, "}\n");
    }
    return b.s;
}

static void compute_metrics(const tvec* tr, double t_target, double* m) { /* pipeline.cpp:325-371 */
    long tokens = 0, cur = 0, matched_sum = 0, matched_n = 0, seg_total = 0, seg_n = 0;
    double clock = 0.0;
    for (long i = 0; i < tr->n; ++i) {
        const trace_t* t = &tr->v[i];
        tokens += t->committed_count;
        clock += t->clock_delta;
        if (t->pending_reject) {
            seg_total += cur + t->accepted_pending; seg_n++;
            cur = t->committed_count - t->accepted_pending;
        } else if (t->rejected) {
            seg_total += cur + t->committed_count; seg_n++;
            cur = 0;
        } else {
            cur += t->committed_count;
        }
        for (long k = 0; k < t->draft_matched.n; ++k) { matched_sum += t->draft_matched.v[k]; matched_n++; }
        if (t->target_matched >= 0) { matched_sum += t->target_matched; matched_n++; }
    }
    if (cur > 0) { seg_total += cur; seg_n++; }
    m[0] = (double)tokens;
    m[1] = (double)tr->n;
    m[2] = clock;
    m[3] = seg_n ? (double)seg_total / (double)seg_n : 0.0;
    m[4] = matched_n ? (double)matched_sum / (double)matched_n : 0.0;
    m[5] = clock > 0.0 ? (double)tokens * t_target / clock : 0.0;
    m[6] = 0.0;
    m[7] = 0.0;
}

static const char* source_name(int s) { /* datastore.cpp:33-42 */
    static const char* names[] = {"prior", "dynamic", "rejected", "context", "miss"};
    return names[s];
}

/* ------------------------------------------------------------------ speculation.cpp / pipeline.cpp */
typedef struct { int vocab; orc_argmax_fn fn; void* user; } model_t;

typedef struct { ivec emitted; int matched, source; } seg_t;

/* accept_with_model, greedy branch (speculation.cpp:7-52): rows[k] = argmax of dists[k] */
static void accept_greedy(const int* rows, const int* cands, int c, int vocab, seg_t* out) {
    int s = 0;
    while (s < c) {
        const int cand = cands[s];
        if (cand < 0 || cand >= vocab) break;
        if (cand != rows[s]) break;
        iv_push(&out->emitted, cand);
        ++s;
    }
    out->matched = s;
    iv_push(&out->emitted, rows[s]); /* correction or continuation: argmax in both greedy cases */
}

static int forward_argmax(const model_t* m, const int* ctx, int L, const int* cands, int c, int* out) {
    if (L <= 0) return fail("forward_batch: empty context");
    if (m->fn(m->user, ctx, L, cands, c, out)) return -1;
    for (int k = 0; k <= c; ++k) if (out[k] < 0) return fail("degenerate distribution");
    return 0;
}

/* retrieval_forward (speculation.cpp:54-66) */
static int retrieval_forward(const model_t* m, orc_store* st, const int* ctx, int L, int depth,
                             int use_retrieval, seg_t* seg) {
    int* cands = (int*)malloc((size_t)(depth > 0 ? depth : 1) * sizeof(int));
    int c = 0, src = ORC_MISS, ord = 0;
    if (use_retrieval && orc_store_lookup(st, ctx, L, depth, cands, &c, &src, &ord)) { free(cands); return -1; }
    int* rows = (int*)malloc((size_t)(c + 1) * sizeof(int));
    int rc = forward_argmax(m, ctx, L, cands, c, rows);
    if (!rc) { accept_greedy(rows, cands, c, m->vocab, seg); seg->source = src; }
    free(rows); free(cands);
    return rc;
}

typedef struct { seg_t* segs; int n_segs; ivec tokens; } chain_t;
static void chain_free(chain_t* ch) {
    for (int i = 0; i < ch->n_segs; ++i) iv_free(&ch->segs[i].emitted);
    free(ch->segs); iv_free(&ch->tokens);
}

/* iterative_draft (speculation.cpp:68-86) */
static int iterative_draft(const model_t* m, orc_store* st, const int* ctx0, int L0, int gamma,
                           int depth, int use_retrieval, chain_t* ch) {
    if (gamma < 1) return fail("iterative_draft: gamma must be >= 1");
    ivec ctx = {0};
    iv_append(&ctx, ctx0, L0);
    ch->segs = (seg_t*)calloc((size_t)gamma, sizeof(seg_t));
    ch->n_segs = gamma;
    for (int j = 0; j < gamma; ++j) {
        if (retrieval_forward(m, st, ctx.v, (int)ctx.n, depth, use_retrieval, &ch->segs[j])) {
            iv_free(&ctx); return -1;
        }
        iv_append(&ctx, ch->segs[j].emitted.v, ch->segs[j].emitted.n);
        iv_append(&ch->tokens, ch->segs[j].emitted.v, ch->segs[j].emitted.n);
    }
    iv_free(&ctx);
    return 0;
}

/* record_accepted_run / record_rejected_run (pipeline.cpp:72-89) */
static int record_run(orc_store* st, int layer, const int* before, long nb, const int* add, long na) {
    if (na <= 0) return 0;
    long pre = layer == ORC_DYNAMIC ? (long)st->max_order - 1 : 3;
    if (pre > nb) pre = nb;
    ivec rec = {0};
    iv_append(&rec, before + nb - pre, pre);
    iv_append(&rec, add, na);
    int rc = orc_store_record(st, layer, rec.v, (int)rec.n);
    iv_free(&rec);
    return rc;
}

typedef struct {
    ivec committed, spec;
    int mode; /* 0 pre_verify, 1 post_verify */
    int prev_tokens;
    long round, last_committed_len;
    double clock;
} state_t;

/* one round: do_draft + do_target + finish_round (pipeline.cpp:39-206, 223-262), serial engine */
static int run_round(state_t* S, const model_t* dm, const model_t* tm, orc_store* st,
                     const orc_opts* o, tvec* traces) {
    /* check_state, pipeline.cpp:208-219 */
    if (S->mode == 0 && S->spec.n) return fail("pre-verify mode with a speculative tail");
    if (S->mode == 1 && S->prev_tokens != S->spec.n) return fail("prev_tokens out of sync with speculative tail");
    int rc = 0;
    ivec ctx = {0};
    iv_append(&ctx, S->committed.v, S->committed.n);
    iv_append(&ctx, S->spec.v, S->spec.n);
    chain_t ch = {0};
    /* do_draft (pipeline.cpp:39-46) */
    if (iterative_draft(dm, st, ctx.v, (int)ctx.n, o->gamma, o->depth, o->draft_retrieval, &ch)) {
        rc = -1; goto out;
    }
    /* do_target (pipeline.cpp:48-70) */
    const int n_spec = (int)S->spec.n;
    int* cands = (int*)malloc((size_t)(o->depth + 1) * sizeof(int));
    int c = 0, src = ORC_MISS, ord = 0;
    if (o->target_retrieval && orc_store_lookup(st, ctx.v, (int)ctx.n, o->depth, cands, &c, &src, &ord)) {
        free(cands); rc = -1; goto out;
    }
    ivec batch = {0};
    iv_append(&batch, S->spec.v, S->spec.n);
    iv_append(&batch, cands, c);
    int* rows = (int*)malloc((size_t)(batch.n + 1) * sizeof(int));
    if (forward_argmax(tm, S->committed.v, (int)S->committed.n, batch.v, (int)batch.n, rows)) {
        free(cands); iv_free(&batch); free(rows); rc = -1; goto out;
    }
    seg_t ext = {0};
    accept_greedy(rows + n_spec, cands, c, tm->vocab, &ext);
    ext.source = src;

    /* finish_round (pipeline.cpp:91-206) */
    trace_t* tr = tv_new(traces);
    tr->round = S->round;
    tr->mode = S->mode ? "post_verify" : "pre_verify";
    tr->pending = n_spec;
    tr->draft_len = (int)ch.tokens.n;
    if (o->draft_retrieval)
        for (int j = 0; j < ch.n_segs; ++j) iv_push(&tr->draft_matched, ch.segs[j].matched);
    tr->target_matched = o->target_retrieval ? ext.matched : -1;
    tr->target_source = source_name(ext.source);

    int rej = -1; /* verify_against_target greedy, verification.cpp:60-78 */
    for (int k = 0; k < n_spec; ++k)
        if (S->spec.v[k] != rows[k]) { rej = k; break; }

    const long nb = S->committed.n;
    ivec add = {0}, new_spec = {0}, pre = {0};
    if (rej >= 0) {
        const int k = rej;
        tr->accepted_pending = k;
        tr->pending_reject = 1;
        tr->rejected = 1;
        tr->kind = "pending_reject";
        iv_append(&add, S->spec.v, k);
        iv_push(&add, rows[k]);
        iv_append(&pre, S->committed.v, nb);
        iv_append(&pre, S->spec.v, k);
        rc |= record_run(st, ORC_REJECTED, pre.v, pre.n, S->spec.v + k, n_spec - k);
        pre.n = 0;
        iv_append(&pre, S->committed.v, nb);
        iv_append(&pre, S->spec.v, n_spec);
        rc |= record_run(st, ORC_REJECTED, pre.v, pre.n, ch.tokens.v, ch.tokens.n);
    } else {
        tr->accepted_pending = n_spec;
        iv_append(&add, S->spec.v, n_spec);
        iv_append(&add, ext.emitted.v, ext.emitted.n);
        const long ne = ext.emitted.n, nf = ch.tokens.n;
        const long cmp = nf < ne ? nf : ne;
        long j = 0;
        while (j < cmp && ch.tokens.v[j] == ext.emitted.v[j]) ++j;
        if (j == ne && nf > ne) {
            tr->kind = "extend_keep_draft";
            iv_append(&new_spec, ch.tokens.v + ne, nf - ne);
        } else if (j == cmp) {
            tr->kind = "extend_draft_subsumed";
        } else {
            tr->kind = "extend_drop_draft";
            tr->rejected = 1;
            iv_append(&pre, S->committed.v, nb);
            iv_append(&pre, S->spec.v, n_spec);
            iv_append(&pre, ch.tokens.v, j);
            rc |= record_run(st, ORC_REJECTED, pre.v, pre.n, ch.tokens.v + j, nf - j);
        }
    }
    tr->committed_count = (int)add.n;
    rc |= record_run(st, ORC_DYNAMIC, S->committed.v, nb, add.v, add.n);
    iv_append(&S->committed, add.v, add.n);
    /* rollback(state, |committed|) (pipeline.cpp:15-30): keep_len == |committed| <= ctx and
     * >= last_committed_len by construction; it clears the speculative tail */
    S->spec.n = 0;
    iv_append(&S->spec, new_spec.v, new_spec.n);
    S->mode = S->spec.n ? 1 : 0;
    S->prev_tokens = S->spec.n ? (int)S->spec.n : o->gamma;
    S->last_committed_len = S->committed.n;
    S->round += 1;
    {
        const double draft_time = o->gamma * (o->t_draft + (o->draft_retrieval ? o->t_lookup : 0.0));
        const double target_time = o->t_target + (o->target_retrieval ? o->t_lookup : 0.0);
        tr->clock_delta = (draft_time > target_time ? draft_time : target_time) + o->t_sync;
        S->clock += tr->clock_delta;
    }
    iv_free(&add); iv_free(&new_spec); iv_free(&pre); iv_free(&ext.emitted);
    free(cands); iv_free(&batch); free(rows);
    if (rc) rc = -1;
out:
    chain_free(&ch);
    iv_free(&ctx);
    return rc;
}

static int finish_output(const ivec* committed, long prompt_len, int max_new, int* out, int cap, int* n_out) {
    long n = committed->n - prompt_len;
    if (n > max_new) n = max_new;
    if (n > cap) return fail("output buffer too small");
    memcpy(out, committed->v + prompt_len, (size_t)n * sizeof(int));
    *n_out = (int)n;
    return 0;
}

int orc_run(int draft_vocab, orc_argmax_fn dfn, void* duser, int target_vocab, orc_argmax_fn tfn,
            void* tuser, orc_store* st, const int* prompt, int n_prompt, int max_new,
            const orc_opts* o, int* out_tokens, int cap, int* n_out, char** jsonl, double* metrics) {
    /* run, pipeline.cpp:264-323 */
    if (max_new < 1) return fail("max_new_tokens must be >= 1");
    if (n_prompt <= 0) return fail("prompt must be nonempty");
    if (o->gamma < 1) return fail("gamma must be >= 1");
    if (o->depth < 1) return fail("depth must be >= 1");
    if (o->t_target < 0.0 || o->t_draft <= 0.0 || o->t_lookup < 0.0 || o->t_sync < 0.0)
        return fail("latency values out of range");
    const model_t dm = {draft_vocab, dfn, duser}, tm = {target_vocab, tfn, tuser};
    const long base_lookups = st->stats[0];
    const long base_hits = st->stats[1] + st->stats[2] + st->stats[3] + st->stats[4];
    state_t S = {0};
    iv_append(&S.committed, prompt, n_prompt);
    S.prev_tokens = o->gamma;
    S.last_committed_len = n_prompt;
    int rc = orc_store_record(st, ORC_DYNAMIC, prompt, n_prompt);
    tvec tr = {0};
    const int eos = target_vocab - 1;
    long scanned = n_prompt;
    int done = 0;
    while (!rc && !done) {
        if (run_round(&S, &dm, &tm, st, o, &tr)) { rc = -1; break; }
        for (; scanned < S.committed.n; ++scanned) {
            if (S.committed.v[scanned] == eos) { S.committed.n = scanned + 1; done = 1; break; }
        }
        if (S.committed.n - n_prompt >= max_new) done = 1;
        if (S.round > 1000000) { rc = fail("round limit exceeded; pipeline stalled"); }
    }
    if (!rc) rc = finish_output(&S.committed, n_prompt, max_new, out_tokens, cap, n_out);
    if (!rc) {
        compute_metrics(&tr, o->t_target, metrics);
        const long lookups = st->stats[0] - base_lookups;
        const long hits = st->stats[1] + st->stats[2] + st->stats[3] + st->stats[4] - base_hits;
        metrics[7] = (double)lookups;
        metrics[6] = lookups ? (double)hits / (double)lookups : 0.0;
        if (jsonl) *jsonl = traces_jsonl(&tr);
        orc_store_flush(st);
    }
    tv_free(&tr);
    iv_free(&S.committed); iv_free(&S.spec);
    return rc;
}

int orc_run_ar(int target_vocab, orc_argmax_fn tfn, void* tuser, const int* prompt, int n_prompt,
               int max_new, double t_target, int* out_tokens, int cap, int* n_out, char** jsonl,
               double* metrics) { /* run_vanilla_ar, harness.cpp:233-258 */
    const model_t tm = {target_vocab, tfn, tuser};
    const int eos = target_vocab - 1;
    ivec ctx = {0};
    iv_append(&ctx, prompt, n_prompt);
    tvec tr = {0};
    int rc = 0;
    for (int i = 0; i < max_new; ++i) {
        int tok;
        if (forward_argmax(&tm, ctx.v, (int)ctx.n, NULL, 0, &tok)) { rc = -1; break; }
        iv_push(&ctx, tok);
        trace_t* t = tv_new(&tr);
        t->round = i; t->mode = "ar"; t->committed_count = 1; t->kind = "ar_step";
        t->clock_delta = t_target;
        if (tok == eos) break;
    }
    if (!rc) rc = finish_output(&ctx, n_prompt, max_new, out_tokens, cap, n_out);
    if (!rc) {
        compute_metrics(&tr, t_target, metrics);
        metrics[2] = metrics[0] * t_target;
        metrics[5] = 1.0;
        if (jsonl) *jsonl = traces_jsonl(&tr);
    }
    tv_free(&tr); iv_free(&ctx);
    return rc;
}

/* run_serial_sd (harness.cpp:264-369), greedy */
static int run_serial_sd(const model_t* dm, const model_t* tm, orc_store* st, const int* prompt,
                         int n_prompt, int max_new, int gamma, int depth, int use_retrieval,
                         double t_target, double t_draft, double t_lookup, double t_sync,
                         int* out_tokens, int cap, int* n_out, char** jsonl, double* metrics) {
    const long base_lookups = st->stats[0];
    const long base_hits = st->stats[1] + st->stats[2] + st->stats[3] + st->stats[4];
    int rc = orc_store_record(st, ORC_DYNAMIC, prompt, n_prompt);
    const int eos = tm->vocab - 1;
    ivec committed = {0};
    iv_append(&committed, prompt, n_prompt);
    tvec tr = {0};
    long round = 0, scanned = n_prompt;
    int done = 0;
    while (!rc && !done) {
        chain_t ch = {0};
        if (iterative_draft(dm, st, committed.v, (int)committed.n, gamma, depth, use_retrieval, &ch)) {
            chain_free(&ch); rc = -1; break;
        }
        int* rows = (int*)malloc((size_t)(ch.tokens.n + 1) * sizeof(int));
        if (forward_argmax(tm, committed.v, (int)committed.n, ch.tokens.v, (int)ch.tokens.n, rows)) {
            free(rows); chain_free(&ch); rc = -1; break;
        }
        int rej = -1;
        for (long k = 0; k < ch.tokens.n; ++k) if (ch.tokens.v[k] != rows[k]) { rej = (int)k; break; }
        trace_t* t = tv_new(&tr);
        t->round = round; t->mode = "serial"; t->draft_len = (int)ch.tokens.n;
        if (use_retrieval) for (int j = 0; j < ch.n_segs; ++j) iv_push(&t->draft_matched, ch.segs[j].matched);
        ivec add = {0};
        if (rej >= 0) {
            t->accepted_pending = rej; t->pending_reject = 1; t->rejected = 1; t->kind = "reject";
            iv_append(&add, ch.tokens.v, rej);
            iv_push(&add, rows[rej]);
            ivec pre = {0};
            iv_append(&pre, committed.v, committed.n);
            iv_append(&pre, ch.tokens.v, rej);
            rc |= record_run(st, ORC_REJECTED, pre.v, pre.n, ch.tokens.v + rej, ch.tokens.n - rej);
            iv_free(&pre);
        } else {
            t->accepted_pending = (int)ch.tokens.n; t->kind = "all_accepted";
            iv_append(&add, ch.tokens.v, ch.tokens.n);
            iv_push(&add, rows[ch.tokens.n]);
        }
        t->committed_count = (int)add.n;
        t->clock_delta = gamma * (t_draft + (use_retrieval ? t_lookup : 0.0)) + t_target + t_sync;
        rc |= record_run(st, ORC_DYNAMIC, committed.v, committed.n, add.v, add.n);
        iv_append(&committed, add.v, add.n);
        iv_free(&add); free(rows); chain_free(&ch);
        ++round;
        for (; scanned < committed.n; ++scanned)
            if (committed.v[scanned] == eos) { committed.n = scanned + 1; done = 1; break; }
        if (committed.n - n_prompt >= max_new) done = 1;
        if (round > 1000000) rc = fail("round limit exceeded; decoder stalled");
    }
    if (!rc) rc = finish_output(&committed, n_prompt, max_new, out_tokens, cap, n_out);
    if (!rc) {
        compute_metrics(&tr, t_target, metrics);
        const long lookups = st->stats[0] - base_lookups;
        const long hits = st->stats[1] + st->stats[2] + st->stats[3] + st->stats[4] - base_hits;
        metrics[7] = (double)lookups;
        metrics[6] = lookups ? (double)hits / (double)lookups : 0.0;
        if (jsonl) *jsonl = traces_jsonl(&tr);
    }
    tv_free(&tr); iv_free(&committed);
    return rc < 0 ? -1 : rc;
}

/* ------------------------------------------------------------------ harness config + setup */
typedef struct {
    int vocab; double rho; int corpus_len, draft_order, target_order; double smoothing;
    double t_target, t_draft, t_lookup, t_sync;
    int gamma, depth, ngram, prior_rounds; double temperature; unsigned long long seed;
    char method[32]; int max_new_tokens, prompt_len, rejected_cache, concurrent;
} cfg_t;

static void trim(char* s) {
    char* a = s;
    while (*a == ' ' || *a == '\t' || *a == '\r') ++a;
    memmove(s, a, strlen(a) + 1);
    long n = (long)strlen(s);
    while (n > 0 && (s[n - 1] == ' ' || s[n - 1] == '\t' || s[n - 1] == '\r')) s[--n] = 0;
}
static int parse_int(const char* v, int* out) { char* e; long x = strtol(v, &e, 10); if (e == v) return -1; *out = (int)x; return 0; }
static int parse_dbl(const char* v, double* out) { char* e; double x = strtod(v, &e); if (e == v) return -1; *out = x; return 0; }

static int parse_config(const char* text, cfg_t* c) { /* harness.cpp:55-114 (+ defaults harness.hpp:21-44) */
    memset(c, 0, sizeof *c);
    c->vocab = 32; c->rho = 0.5; c->corpus_len = 4096; c->draft_order = 1; c->target_order = 2;
    c->smoothing = 0.1; c->t_target = 1.0; c->t_draft = 0.25; c->gamma = 0; c->depth = 10;
    c->ngram = 3; c->prior_rounds = 10; c->seed = 1; strcpy(c->method, "double");
    c->max_new_tokens = 256; c->prompt_len = 8; c->rejected_cache = 1;
    char* dup = strdup(text);
    char* save = NULL;
    int rc = 0;
    for (char* line = strtok_r(dup, "\n", &save); line && !rc; line = strtok_r(NULL, "\n", &save)) {
        char* h = strchr(line, '#');
        if (h) *h = 0;
        char* eq = strchr(line, '=');
        if (!eq) {
            char t[512]; snprintf(t, sizeof t, "%s", line); trim(t);
            if (*t) rc = fail("config: expected key=value");
            continue;
        }
        *eq = 0;
        char key[128], val[256];
        snprintf(key, sizeof key, "%s", line); snprintf(val, sizeof val, "%s", eq + 1);
        trim(key); trim(val);
        int bad = 0;
        if (!strcmp(key, "vocab")) bad = parse_int(val, &c->vocab);
        else if (!strcmp(key, "rho")) bad = parse_dbl(val, &c->rho);
        else if (!strcmp(key, "corpus_len")) bad = parse_int(val, &c->corpus_len);
        else if (!strcmp(key, "draft_order")) bad = parse_int(val, &c->draft_order);
        else if (!strcmp(key, "target_order")) bad = parse_int(val, &c->target_order);
        else if (!strcmp(key, "smoothing")) bad = parse_dbl(val, &c->smoothing);
        else if (!strcmp(key, "t_target")) bad = parse_dbl(val, &c->t_target);
        else if (!strcmp(key, "t_draft")) bad = parse_dbl(val, &c->t_draft);
        else if (!strcmp(key, "t_lookup")) bad = parse_dbl(val, &c->t_lookup);
        else if (!strcmp(key, "t_sync")) bad = parse_dbl(val, &c->t_sync);
        else if (!strcmp(key, "gamma")) bad = parse_int(val, &c->gamma);
        else if (!strcmp(key, "depth")) bad = parse_int(val, &c->depth);
        else if (!strcmp(key, "ngram")) bad = parse_int(val, &c->ngram);
        else if (!strcmp(key, "prior_rounds")) bad = parse_int(val, &c->prior_rounds);
        else if (!strcmp(key, "temperature")) bad = parse_dbl(val, &c->temperature);
        else if (!strcmp(key, "seed")) { char* e; c->seed = strtoull(val, &e, 10); bad = e == val; }
        else if (!strcmp(key, "method")) snprintf(c->method, sizeof c->method, "%s", val);
        else if (!strcmp(key, "max_new_tokens")) bad = parse_int(val, &c->max_new_tokens);
        else if (!strcmp(key, "prompt_len")) bad = parse_int(val, &c->prompt_len);
        else if (!strcmp(key, "rejected_cache")) c->rejected_cache = !strcmp(val, "1") || !strcmp(val, "true");
        else if (!strcmp(key, "engine")) {
            if (!strcmp(val, "serial")) c->concurrent = 0;
            else if (!strcmp(val, "concurrent")) c->concurrent = 1;
            else bad = 1;
        } else rc = fail("config: unknown key");
        if (bad) rc = fail("config: bad value");
    }
    free(dup);
    if (rc) return rc;
    /* ExperimentConfig::validate, harness.cpp:37-53 */
    if (c->vocab < 4) return fail("vocab must be >= 4");
    if (c->rho < 0.0 || c->rho > 1.0) return fail("rho out of [0,1]");
    if (c->corpus_len < c->prompt_len + 1) return fail("corpus too short");
    if (c->draft_order < 1 || c->target_order < 1) return fail("model orders must be >= 1");
    if (c->smoothing < 0.0) return fail("smoothing must be >= 0");
    if (c->t_target < 0.0 || c->t_draft <= 0.0 || c->t_lookup < 0.0 || c->t_sync < 0.0)
        return fail("latency values out of range");
    if (c->gamma < 0) return fail("gamma must be >= 0");
    if (c->depth < 1) return fail("depth must be >= 1");
    if (c->ngram < 1) return fail("ngram must be >= 1");
    if (c->prior_rounds < 0) return fail("prior_rounds must be >= 0");
    if (c->temperature != 0.0) return fail("oracle restatement covers greedy (temperature 0) only");
    if (c->max_new_tokens < 1) return fail("max_new_tokens must be >= 1");
    if (c->prompt_len < 1) return fail("prompt_len must be >= 1");
    return 0;
}

int orc_run_config(const char* cfg_text, const char* method, int* out_tokens, int cap, int* n_out,
                   char** jsonl, double* metrics) { /* run_method_on, harness.cpp:403-429 */
    cfg_t c;
    if (parse_config(cfg_text, &c)) return -1;
    const char* m = method ? method : c.method;
    int* toks = (int*)malloc((size_t)c.corpus_len * sizeof(int));
    int* lens = (int*)malloc((size_t)(c.corpus_len / 64 + 2) * sizeof(int));
    int nseq = 0, rc = 0;
    orc_table *dt = NULL, *tt = NULL;
    orc_store* st = NULL;
    if (orc_gen_corpus(c.vocab, c.rho, c.corpus_len, c.seed, toks, lens, &nseq)) { rc = -1; goto done; }
    dt = orc_table_build(toks, lens, nseq, c.draft_order, c.smoothing, c.vocab);
    tt = orc_table_build(toks, lens, nseq, c.target_order, c.smoothing, c.vocab);
    if (!dt || !tt) { rc = -1; goto done; }
    if (lens[0] < c.prompt_len) { rc = fail("prompt_len exceeds the first corpus sequence"); goto done; }
    const int gamma = c.gamma > 0 ? c.gamma : (int)ceil(c.t_target / c.t_draft); /* :32-35 */
    st = orc_store_new(c.ngram, c.depth); /* build_store, harness.cpp:204-210 */
    {
        long at = 0;
        for (int i = 0; i < nseq && i < c.prior_rounds; ++i) { /* build_prior, datastore.cpp:149-159 */
            orc_layer_insert(st, ORC_PRIOR, toks + at, lens[i], i);
            at += lens[i];
        }
    }
    st->rejected_enabled = c.rejected_cache;
    if (!strcmp(m, "vanilla_ar")) {
        rc = orc_run_ar(c.vocab, orc_table_argmax_rows, tt, toks, c.prompt_len, c.max_new_tokens,
                        c.t_target, out_tokens, cap, n_out, jsonl, metrics);
    } else if (!strcmp(m, "sd") || !strcmp(m, "draft_retrieval")) {
        const model_t dm = {c.vocab, orc_table_argmax_rows, dt}, tm = {c.vocab, orc_table_argmax_rows, tt};
        rc = run_serial_sd(&dm, &tm, st, toks, c.prompt_len, c.max_new_tokens, gamma, c.depth,
                           !strcmp(m, "draft_retrieval"), c.t_target, c.t_draft, c.t_lookup,
                           c.t_sync, out_tokens, cap, n_out, jsonl, metrics);
    } else {
        orc_opts o = {gamma, c.depth, 1, 1, c.t_target, c.t_draft, c.t_lookup, c.t_sync};
        if (!strcmp(m, "psd")) { o.draft_retrieval = 0; o.target_retrieval = 0; }
        else if (!strcmp(m, "target_retrieval")) { o.draft_retrieval = 0; }
        else if (strcmp(m, "double")) { rc = fail("unknown method"); goto done; }
        rc = orc_run(c.vocab, orc_table_argmax_rows, dt, c.vocab, orc_table_argmax_rows, tt, st,
                     toks, c.prompt_len, c.max_new_tokens, &o, out_tokens, cap, n_out, jsonl, metrics);
    }
done:
    orc_table_free(dt); orc_table_free(tt); orc_store_free(st);
    free(toks); free(lens);
    return rc;
}

/* ------------------------------------------------------------------ replay models (bench only) */
typedef struct { int matched; int off; } rseg;
typedef struct { int seg0, nseg, n_spec, rej, corr, ext_m, ext_off; } rround;
struct orc_replay {
    int* data; long len;
    rround* rounds; long n_rounds;
    rseg* segs; long n_segs;
    long dr, ds, tr; /* cursors: draft round/seg, target round */
};

orc_replay* orc_replay_new(const int* log, long len) {
    orc_replay* r = (orc_replay*)calloc(1, sizeof *r);
    r->data = (int*)malloc((size_t)(len ? len : 1) * sizeof(int));
    memcpy(r->data, log, (size_t)len * sizeof(int));
    r->len = len;
    long cap_r = 64, cap_s = 256, at = 0;
    r->rounds = (rround*)malloc((size_t)cap_r * sizeof(rround));
    r->segs = (rseg*)malloc((size_t)cap_s * sizeof(rseg));
    while (at < len) {
        if (r->n_rounds == cap_r) { cap_r *= 2; r->rounds = (rround*)realloc(r->rounds, (size_t)cap_r * sizeof(rround)); }
        rround* rd = &r->rounds[r->n_rounds++];
        rd->nseg = log[at++];
        rd->seg0 = (int)r->n_segs;
        for (int j = 0; j < rd->nseg; ++j) {
            if (r->n_segs == cap_s) { cap_s *= 2; r->segs = (rseg*)realloc(r->segs, (size_t)cap_s * sizeof(rseg)); }
            rseg* sg = &r->segs[r->n_segs++];
            sg->matched = log[at++];
            sg->off = (int)at;
            at += sg->matched + 1;
        }
        rd->n_spec = log[at++];
        rd->rej = log[at++];
        rd->corr = log[at++];
        rd->ext_m = log[at++];
        rd->ext_off = (int)at;
        at += rd->ext_m + 1;
    }
    return r;
}
void orc_replay_free(orc_replay* r) {
    if (!r) return;
    free(r->data); free(r->rounds); free(r->segs); free(r);
}
void orc_replay_reset(orc_replay* r) { r->dr = r->ds = r->tr = 0; }

int orc_replay_draft(void* user, const int* ctx, int L, const int* cands, int c, int* out) {
    (void)ctx; (void)L;
    orc_replay* r = (orc_replay*)user;
    while (r->dr < r->n_rounds && r->ds >= r->rounds[r->dr].nseg) { r->dr++; r->ds = 0; }
    if (r->dr >= r->n_rounds) return fail("replay: draft log exhausted");
    const rseg* sg = &r->segs[r->rounds[r->dr].seg0 + r->ds++];
    const int m = sg->matched;
    const int e = r->data[sg->off + m];
    for (int s = 0; s <= c; ++s) out[s] = s < m ? cands[s] : e;
    return 0;
}

int orc_replay_target(void* user, const int* ctx, int L, const int* cands, int c, int* out) {
    (void)ctx; (void)L;
    orc_replay* r = (orc_replay*)user;
    if (r->tr >= r->n_rounds) return fail("replay: target log exhausted");
    const rround* rd = &r->rounds[r->tr++];
    for (int k = 0; k < rd->n_spec && k <= c; ++k)
        out[k] = (rd->rej < 0 || k < rd->rej) ? cands[k] : rd->corr;
    const int e = r->data[rd->ext_off + rd->ext_m];
    for (int s = 0; rd->n_spec + s <= c; ++s)
        out[rd->n_spec + s] = s < rd->ext_m ? cands[rd->n_spec + s] : e;
    return 0;
}


/* ===================================================================== verifier (T >= 0)
 * verification.cpp:19-132.  Rows are ragged like ProbVector: row r = probs[off[r] .. off[r+1]).
 * Errors: -1 std::invalid_argument, -2 std::runtime_error (message in orc_last_error()). */
int orc_accept_prob(const double* p, int np, const double* q, int nq, int x, double* out) { /* :19-23 */
    if (x < 0 || x >= nq || x >= np) { (void)fail("token out of range"); return -1; }
    if (q[x] <= 0.0) { (void)fail("draft mass zero on emitted token"); return -1; }
    *out = p[x] / q[x] < 1.0 ? p[x] / q[x] : 1.0;
    return 0;
}

static int orc_sample_from(const double* w, int n, double total, orc_mt64* g) { /* :25-38 */
    const double u = orc_uniform(g) * total;
    double acc = 0.0;
    int last = -1;
    for (int i = 0; i < n; ++i) {
        if (w[i] <= 0.0) continue;
        last = i;
        acc += w[i];
        if (u < acc) return last;
    }
    return last;
}

int orc_residual_sample(const double* p, int np, const double* q, int nq, orc_mt64* g, int* out) { /* :40-50 */
    if (nq < np) { (void)fail("residual: q shorter than p"); return -1; }
    double* res = (double*)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1));
    double total = 0.0;
    for (int i = 0; i < np; ++i) {
        res[i] = p[i] - q[i] > 0.0 ? p[i] - q[i] : 0.0;
        total += res[i];
    }
    if (total <= 0.0) { free(res); (void)fail("residual distribution is zero"); return -2; }
    *out = orc_sample_from(res, np, total, g);
    free(res);
    return 0;
}

int orc_residual_point_mass(const double* p, int np, int x, orc_mt64* g, int* out) { /* :52-58 */
    if (x < 0 || x >= np) { (void)fail("token out of range"); return -1; }
    double* res = (double*)malloc(sizeof(double) * (size_t)np);
    double total = 0.0;
    for (int i = 0; i < np; ++i) res[i] = i == x ? 0.0 : p[i];
    for (int i = 0; i < np; ++i) total += res[i];
    if (total <= 0.0) { free(res); (void)fail("residual distribution is zero"); return -2; }
    *out = orc_sample_from(res, np, total, g);
    free(res);
    return 0;
}

int orc_verify_against_target(const int* draft, int n_draft, const double* dp, const int64_t* doff, int n_dp,
                              const double* tp, const int64_t* toff, int n_tp, double temperature, orc_mt64* g,
                              int* first_reject) { /* :60-78 */
    *first_reject = -1;
    if (n_tp < n_draft) { (void)fail("target_probs does not cover the draft slice"); return -1; }
    for (int k = 0; k < n_draft; ++k) {
        if (temperature == 0.0) {
            const int a = orc_argmax(tp + toff[k], (int)(toff[k + 1] - toff[k]));
            if (a < 0) { (void)fail("degenerate distribution"); return -2; }
            if (draft[k] != a) { *first_reject = k; return 0; }
        } else {
            double a;
            if (k >= n_dp) { (void)fail("draft_probs does not cover the draft slice"); return -1; }
            const int rc = orc_accept_prob(tp + toff[k], (int)(toff[k + 1] - toff[k]), dp + doff[k],
                                           (int)(doff[k + 1] - doff[k]), draft[k], &a);
            if (rc) return rc;
            if (orc_uniform(g) >= a) { *first_reject = k; return 0; }
        }
    }
    return 0;
}

int orc_guided_output(const int* draft, int n_draft, const double* dp, const int64_t* doff, int n_dp,
                      const int* gtok, int n_gtok, const double* gp, const int64_t* goff, int n_gp,
                      int first_reject, double temperature, orc_mt64* g, int* committed, int cap,
                      int* n_committed, int* accepted_len, int* kind) { /* :80-132 */
    int n = 0;
#define ORC_PUSH(t) do { if (n < cap) committed[n] = (t); ++n; } while (0)
    if (first_reject < 0) {
        *accepted_len = n_draft;
        for (int i = 0; i < n_draft; ++i) ORC_PUSH(draft[i]);
        *kind = 0; /* AllAccepted */
        int covers = temperature == 0.0 && n_gtok > n_draft;
        for (int i = 0; covers && i < n_draft; ++i) covers = draft[i] == gtok[i];
        if (covers) {
            for (int i = n_draft; i < n_gtok; ++i) ORC_PUSH(gtok[i]);
            *kind = 2; /* Extension */
        }
        *n_committed = n;
        return 0;
    }
    const int i = first_reject;
    if (i > n_draft) { (void)fail("reject index past the draft slice"); return -1; }
    *accepted_len = i;
    for (int k = 0; k < i; ++k) ORC_PUSH(draft[k]);
    if (temperature == 0.0) {
        if (i < n_gtok) {
            for (int k = i; k < n_gtok; ++k) ORC_PUSH(gtok[k]);
        } else if (i < n_gp) {
            const int a = orc_argmax(gp + goff[i], (int)(goff[i + 1] - goff[i]));
            if (a < 0) { (void)fail("degenerate distribution"); return -2; }
            ORC_PUSH(a);
        } else {
            (void)fail("guided_output: reject position uncovered");
            return -1;
        }
        *kind = 1; /* Correction */
        *n_committed = n;
        return 0;
    }
    if (i >= n_gp) { (void)fail("guided_output: reject position uncovered"); return -1; }
    if (i >= n_dp) { (void)fail("draft_probs does not cover the reject position"); return -1; }
    int t;
    const int rc = orc_residual_sample(gp + goff[i], (int)(goff[i + 1] - goff[i]), dp + doff[i],
                                       (int)(doff[i + 1] - doff[i]), g, &t);
    if (rc) return rc;
    ORC_PUSH(t);
    *kind = 3; /* ResidualCorrection */
    *n_committed = n;
#undef ORC_PUSH
    return 0;
}
