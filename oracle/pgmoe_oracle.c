/*
 * pgmoe_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference `moesim` pre-gated MoE math
 * (/root/reference/pkg/src/moesim/{rng,linalg,core}.py) used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg.  The product path (paper_2308_12066_b200/) never links or calls it.
 *
 * Arithmetic contract (compile with -O2 -ffp-contract=off, no -ffast-math):
 *   - every product is a separately rounded fp64 multiply (no FMA), as in
 *     CPython float arithmetic;
 *   - matvec_columns (gate logits) is a plain left-to-right serial sum
 *     starting from 0.0 (linalg.py:25-38);
 *   - matvec and the softmax normalizer use CPython >= 3.12 builtin sum(),
 *     i.e. Neumaier-compensated summation with the final "add c if finite"
 *     step (linalg.py:20-22, linalg.py:54-59 executed on Python 3.12);
 *   - exp is the C library exp(), which is what math.exp calls.
 * Pinned against the reference itself: the JSON fixtures under tests/golden are produced by
 * tests/golden/gen_golden.py importing moesim, and tests/test_oracle.py
 * checks this file bit-for-bit against them.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OG_OK 0
#define OG_E_CONFIG 1
#define OG_E_SHAPE 2
#define OG_E_GATE_OVERFLOW 3
#define OG_E_GATE_UNDERFLOW 4
#define OG_E_ROUTING 5

#define DT_F32 0
#define DT_BF16 1
#define DT_F64 2

/* ------------------------------------------------------------------ rng.py */

static const uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;

/* rng.py:15-18 (_mix64) */
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.py:21-31 (SplitMix64.next_u64) — n draws from `seed`. */
void og_splitmix64(uint64_t seed, int n, uint64_t *out) {
    uint64_t s = seed;
    for (int i = 0; i < n; ++i) {
        s += GOLDEN;
        out[i] = mix64(s);
    }
}

/* rng.py:34-40 (derive_seed) — tags are reduced mod 2^64 (tag -1 -> 2^64-1). */
uint64_t og_derive_seed(uint64_t base, const int64_t *tags, int ntags) {
    uint64_t x = base;
    for (int i = 0; i < ntags; ++i) {
        x = mix64(x + GOLDEN);
        x = mix64(x ^ (uint64_t)tags[i]);
    }
    return x;
}

typedef struct { uint64_t s[4]; } xo_t;

/* rng.py:46-48 (state from four SplitMix64 draws) */
static void xo_init(xo_t *g, uint64_t seed) { og_splitmix64(seed, 4, g->s); }

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.py:50-62 (Xoshiro256StarStar.next_u64) */
static inline uint64_t xo_next(xo_t *g) {
    uint64_t *s = g->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

void og_xoshiro_u64(uint64_t seed, int n, uint64_t *out) {
    xo_t g;
    xo_init(&g, seed);
    for (int i = 0; i < n; ++i) out[i] = xo_next(&g);
}

/* rng.py:70-88 (fill): lo + span*((r>>11)*2^-53), each op rounded. */
void og_fill(uint64_t seed, size_t n, double lo, double hi, double *out) {
    xo_t g;
    xo_init(&g, seed);
    volatile double span = hi - lo;
    const double to_unit = 0x1p-53;
    for (size_t i = 0; i < n; ++i) {
        double u = (double)(xo_next(&g) >> 11) * to_unit;
        double prod = span * u;
        out[i] = lo + prod;
    }
}

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

static inline double bf16_to_f64(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* Weight matrix of the reference (core.py:200-211) rounded to storage
 * precision: fp64 fill -> fp32 (RNE, as model_io.save_model does,
 * model_io.py:39-60) -> optionally bf16 (RNE of the fp32 value). */
void og_fill_weights(uint64_t seed, size_t n, int dtype, void *out) {
    xo_t g;
    xo_init(&g, seed);
    volatile double span = 0.1 - (-0.1);
    const double to_unit = 0x1p-53;
    for (size_t i = 0; i < n; ++i) {
        double u = (double)(xo_next(&g) >> 11) * to_unit;
        double prod = span * u;
        double v = -0.1 + prod;
        float f = (float)v;
        if (dtype == DT_BF16) ((uint16_t *)out)[i] = f32_to_bf16_rne(f);
        else if (dtype == DT_F32) ((float *)out)[i] = f;
        else ((double *)out)[i] = v;
    }
}

/* ---------------------------------------------------------------- linalg.py */

static inline double wget(const void *p, size_t i, int dt) {
    if (dt == DT_F32) return (double)((const float *)p)[i];
    if (dt == DT_BF16) return bf16_to_f64(((const uint16_t *)p)[i]);
    return ((const double *)p)[i];
}

/* CPython >= 3.12 builtin sum(iterable, 0.0) over floats (Neumaier). */
typedef struct { double s, c; } nsum_t;
static inline void nsum_add(nsum_t *a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}
static inline double nsum_result(const nsum_t *a) {
    double r = a->s;
    if (a->c != 0.0 && isfinite(a->c)) r += a->c;
    return r;
}

double og_pysum(const double *v, size_t n) {
    nsum_t a = {0.0, 0.0};
    for (size_t i = 0; i < n; ++i) nsum_add(&a, v[i]);
    return nsum_result(&a);
}

/* linalg.py:20-22 matvec: rows(W) . x, W row-major [rows][cols]. */
void og_matvec(const void *W, int dt, int rows, int cols, const double *x, double *y) {
    for (int r = 0; r < rows; ++r) {
        nsum_t a = {0.0, 0.0};
        size_t base = (size_t)r * cols;
        for (int c = 0; c < cols; ++c) {
            double p = wget(W, base + c, dt) * x[c];
            nsum_add(&a, p);
        }
        y[r] = nsum_result(&a);
    }
}

/* linalg.py:25-38 matvec_columns: W^T x, ascending-row serial order. */
void og_matvec_columns(const void *W, int dt, int rows, int cols, const double *x, double *out) {
    for (int j = 0; j < cols; ++j) out[j] = 0.0;
    for (int i = 0; i < rows; ++i) {
        double xi = x[i];
        size_t base = (size_t)i * cols;
        for (int j = 0; j < cols; ++j) {
            double p = xi * wget(W, base + j, dt);
            out[j] = out[j] + p;
        }
    }
}

/* linalg.py:54-59 softmax (max-subtract, exp, compensated total, divide). */
void og_softmax(const double *logits, int n, double *probs) {
    double m = logits[0];
    for (int i = 1; i < n; ++i)
        if (logits[i] > m) m = logits[i];
    nsum_t a = {0.0, 0.0};
    for (int i = 0; i < n; ++i) {
        probs[i] = exp(logits[i] - m);
        nsum_add(&a, probs[i]);
    }
    double total = nsum_result(&a);
    for (int i = 0; i < n; ++i) probs[i] = probs[i] / total;
}

/* ------------------------------------------------------------------ core.py */

/* core.py:284-305 gate_forward.  logits_out / probs_out may be NULL. */
int og_gate(const double *x, int d, const void *G, int dt, int E, int k,
            int *ids, double *weights, double *logits_out) {
    if (k > E) return OG_E_CONFIG;
    double *logits = (double *)malloc(sizeof(double) * (size_t)E * 2);
    double *probs = logits + E;
    og_matvec_columns(G, dt, d, E, x, logits);
    for (int j = 0; j < E; ++j)
        if (!isfinite(logits[j])) { free(logits); return OG_E_GATE_OVERFLOW; }
    og_softmax(logits, E, probs);
    /* sorted(range(E), key=(-logit, j))[:k] — selection, k passes. */
    unsigned char *taken = (unsigned char *)calloc((size_t)E, 1);
    for (int s = 0; s < k; ++s) {
        int best = -1;
        for (int j = 0; j < E; ++j) {
            if (taken[j]) continue;
            if (best < 0 || logits[j] > logits[best]) best = j;
        }
        taken[best] = 1;
        ids[s] = best;
        weights[s] = probs[best];
    }
    free(taken);
    if (logits_out) memcpy(logits_out, logits, sizeof(double) * (size_t)E);
    free(logits);
    for (int s = 0; s < k; ++s)
        if (weights[s] <= 0.0) return OG_E_GATE_UNDERFLOW;
    return OG_OK;
}

/* core.py:308-316 expert_forward: y = W2 . relu(W1 . x). */
void og_expert(const double *x, int d, int f, const void *w1, const void *w2, int dt, double *y) {
    double *h = (double *)malloc(sizeof(double) * (size_t)f);
    og_matvec(w1, dt, f, d, x, h);
    for (int i = 0; i < f; ++i) h[i] = h[i] > 0.0 ? h[i] : 0.0; /* linalg.py:41-42 */
    og_matvec(w2, dt, d, f, h, y);
    free(h);
}

/* core.py:319-339 moe_block_forward with routing_in given (k experts):
 * experts in routing order, weighted_sum (linalg.py:45-51), dense matvec.
 * `experts_w1[s]`, `experts_w2[s]` are the weights of ids_in[s]. */
void og_block_experts_dense(const double *x, int d, int f, int k,
                            const void *const *experts_w1, const void *const *experts_w2,
                            const double *w_in, const void *dense, int dt,
                            double *mix_out, double *y) {
    double *mix = mix_out ? mix_out : (double *)malloc(sizeof(double) * (size_t)d);
    double *ey = (double *)malloc(sizeof(double) * (size_t)d);
    for (int i = 0; i < d; ++i) mix[i] = 0.0;
    for (int s = 0; s < k; ++s) {
        og_expert(x, d, f, experts_w1[s], experts_w2[s], dt, ey);
        for (int i = 0; i < d; ++i) {
            double p = w_in[s] * ey[i];
            mix[i] = mix[i] + p;
        }
    }
    og_matvec(dense, dt, d, d, mix, y);
    free(ey);
    if (!mix_out) free(mix);
}

/* Batched extension (not in the reference): per-expert
 * histogram, exclusive scan, stable permutation grouped by ascending expert
 * with ascending (t, s) inside each group, active list ascending. */
void og_permute(const int *ids, int T, int k, int E, int *hist, int *off,
                int *perm, int *act, int *n_act) {
    for (int e = 0; e < E; ++e) hist[e] = 0;
    for (int i = 0; i < T * k; ++i) hist[ids[i]]++;
    off[0] = 0;
    for (int e = 0; e < E; ++e) off[e + 1] = off[e] + hist[e];
    int *cur = (int *)malloc(sizeof(int) * (size_t)E);
    for (int e = 0; e < E; ++e) cur[e] = off[e];
    for (int i = 0; i < T * k; ++i) perm[cur[ids[i]]++] = i;
    free(cur);
    int na = 0;
    for (int e = 0; e < E; ++e)
        if (hist[e] > 0) act[na++] = e;
    *n_act = na;
}

/* ------------------------------------------------- threaded batch helpers */

typedef struct {
    int t0, t1, d, E, k, dt;
    const double *x;
    const void *G;
    int *ids;
    double *w;
    int *status;
} gate_job_t;

static void *gate_worker(void *arg) {
    gate_job_t *j = (gate_job_t *)arg;
    for (int t = j->t0; t < j->t1; ++t) {
        int st = og_gate(j->x + (size_t)t * j->d, j->d, j->G, j->dt, j->E, j->k,
                         j->ids + (size_t)t * j->k, j->w + (size_t)t * j->k, NULL);
        if (st && !*j->status) *j->status = st;
    }
    return NULL;
}

/* gate_forward over T tokens (x row-major [T][d]) on `nthreads` threads. */
int og_gate_batch(const double *x, int T, int d, const void *G, int dt, int E, int k,
                  int *ids, double *w, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > T) nthreads = T > 0 ? T : 1;
    pthread_t th[256];
    gate_job_t jobs[256];
    int status = 0;
    if (nthreads > 256) nthreads = 256;
    for (int i = 0; i < nthreads; ++i) {
        jobs[i] = (gate_job_t){T * i / nthreads, T * (i + 1) / nthreads, d, E, k, dt, x, G, ids, w, &status};
        pthread_create(&th[i], NULL, gate_worker, &jobs[i]);
    }
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    return status;
}

typedef struct {
    int t0, t1, d, f, k, dt;
    const double *x;
    const int *ids;
    const double *w;
    const void *const *w1_of; /* indexed by expert id */
    const void *const *w2_of;
    const void *dense;
    double *y;
} blk_job_t;

static void *blk_worker(void *arg) {
    blk_job_t *j = (blk_job_t *)arg;
    const void *p1[64], *p2[64];
    for (int t = j->t0; t < j->t1; ++t) {
        for (int s = 0; s < j->k; ++s) {
            int e = j->ids[(size_t)t * j->k + s];
            p1[s] = j->w1_of[e];
            p2[s] = j->w2_of[e];
        }
        og_block_experts_dense(j->x + (size_t)t * j->d, j->d, j->f, j->k, p1, p2,
                               j->w + (size_t)t * j->k, j->dense, j->dt, NULL,
                               j->y + (size_t)t * j->d);
    }
    return NULL;
}

/* Experts + combine + dense for T tokens given their routing (ids/w [T][k]).
 * w1_of[e]/w2_of[e]: expert e's matrices (only routed ones are touched). */
int og_block_batch(const double *x, int T, int d, int f, int k,
                   const int *ids, const double *w,
                   const void *const *w1_of, const void *const *w2_of,
                   const void *dense, int dt, double *y, int nthreads) {
    if (k > 64) return OG_E_CONFIG;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > T) nthreads = T > 0 ? T : 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    blk_job_t jobs[256];
    for (int i = 0; i < nthreads; ++i) {
        jobs[i] = (blk_job_t){T * i / nthreads, T * (i + 1) / nthreads, d, f, k, dt,
                              x, ids, w, w1_of, w2_of, dense, y};
        pthread_create(&th[i], NULL, blk_worker, &jobs[i]);
    }
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    return OG_OK;
}
