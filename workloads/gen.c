/*
 * gen.c -- seeded synthetic-input generators shared by the oracle and the
 * CUDA path (the only code both sides use; it holds none of the method's
 * arithmetic).  Recipes: DESIGN.md "Input recipe", BASELINE.json configs.
 *
 * Every row r of a sparse matrix is generated from its own counter-based
 * stream keyed by (seed, purpose, r), so any row range can be produced
 * independently (a rank of a row-partitioned run generates only its rows)
 * and the result does not depend on the thread count.
 *
 * Column indices are distinct and sorted within each row.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;

static inline rng_t rng_for(uint64_t seed, uint64_t purpose, uint64_t row) {
    rng_t r;
    r.s = mix64(seed * 0x9E3779B97F4A7C15ULL + mix64(purpose + 0x632BE59BD9B4E019ULL) +
                mix64(row ^ 0xA0761D6478BD642FULL));
    return r;
}
static inline uint64_t rng_next(rng_t *r) {
    r->s += 0x9E3779B97F4A7C15ULL;
    return mix64(r->s);
}
/* uniform in [0,1) with 53 random bits */
static inline double rng_u01(rng_t *r) {
    return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
}
/* uniform integer in [0, n) (multiply-shift; bias < 2^-40 for n < 2^24) */
static inline int64_t rng_below(rng_t *r, int64_t n) {
    return (int64_t)(((unsigned __int128)rng_next(r) * (unsigned __int128)(uint64_t)n) >> 64);
}
static inline double rng_normal(rng_t *r) {
    double u1 = rng_u01(r), u2 = rng_u01(r);
    if (u1 < 1e-300) u1 = 1e-300;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

enum { PURPOSE_DEG = 1, PURPOSE_COLS = 2, PURPOSE_VALS = 3 };
enum { VAL_NORMAL = 0, VAL_U01 = 1, VAL_UPM1 = 2 };
enum { ROW_UNIFORM = 0, ROW_BANDED = 1 };

/* Zipf(alpha = 2) on {1, 2, ...} by Devroye's rejection method. */
static int64_t zipf2(rng_t *r) {
    for (;;) {
        double u = 1.0 - rng_u01(r); /* (0, 1] */
        double v = rng_u01(r);
        double x = floor(1.0 / u);
        if (x > 9.0e15) continue;
        double t = 1.0 + 1.0 / x;
        /* accept if v * x * (t - 1) / (b - 1) <= t / b with b = 2 */
        if (v * x * (t - 1.0) <= t / 2.0) return (int64_t)x;
    }
}

/* X_r ~ Zipf(2) for rows [r0, r1) */
void wl_zipf2(uint64_t seed, int64_t r0, int64_t r1, int64_t *out) {
    for (int64_t r = r0; r < r1; r++) {
        rng_t g = rng_for(seed, PURPOSE_DEG, (uint64_t)r);
        out[r - r0] = zipf2(&g);
    }
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* d distinct sorted integers uniform in [lo, hi) not in `excl` (sorted,
 * nexcl entries), written to out. */
static void distinct_in_range(rng_t *g, int64_t lo, int64_t hi, int64_t d,
                              const int32_t *excl, int64_t nexcl, int32_t *out) {
    int64_t span = hi - lo;
    if (d <= 0) return;
    if (2 * (d + nexcl) >= span) {
        /* selection sampling (Knuth alg. S) over the non-excluded values */
        int64_t avail = span - nexcl, need = d, e = 0, c = 0;
        for (int64_t v = lo; v < hi && need > 0; v++) {
            while (e < nexcl && excl[e] < v) e++;
            if (e < nexcl && excl[e] == v) continue;
            if ((double)rng_below(g, avail) < (double)need) out[c++] = (int32_t)v, need--;
            avail--;
        }
        return;
    }
    int64_t have = 0;
    while (have < d) {
        for (int64_t i = have; i < d; i++) out[i] = (int32_t)(lo + rng_below(g, span));
        qsort(out, (size_t)d, sizeof(int32_t), cmp_i32);
        /* dedupe and drop excluded values */
        int64_t w = 0, e = 0;
        for (int64_t i = 0; i < d; i++) {
            if (w > 0 && out[w - 1] == out[i]) continue;
            while (e < nexcl && excl[e] < out[i]) e++;
            if (e < nexcl && excl[e] == out[i]) continue;
            out[w++] = out[i];
        }
        have = w;
    }
}

typedef struct {
    int kind, val_kind;
    int64_t m, n, r0, r1, band;
    uint64_t seed;
    const int64_t *row_ptr; /* global row pointer; entries for rows r0..r1 */
    int64_t base;           /* row_ptr[r0] (offset of this range in col/val) */
    int32_t *col;
    double *val;
    int64_t chunk_lo, chunk_hi;
} fill_job;

static void fill_rows(const fill_job *J, int64_t lo, int64_t hi) {
    int32_t *excl = NULL;
    for (int64_t r = lo; r < hi; r++) {
        int64_t p0 = J->row_ptr[r] - J->base, d = J->row_ptr[r + 1] - J->row_ptr[r];
        int32_t *c = J->col + p0;
        rng_t g = rng_for(J->seed, PURPOSE_COLS, (uint64_t)r);
        if (J->kind == ROW_UNIFORM) {
            distinct_in_range(&g, 0, J->n, d, NULL, 0, c);
        } else {
            /* banded-plus-random: half within +-band of the scaled diagonal */
            int64_t cr = (int64_t)((double)r * (double)J->n / (double)J->m);
            int64_t blo = cr - J->band < 0 ? 0 : cr - J->band;
            int64_t bhi = cr + J->band + 1 > J->n ? J->n : cr + J->band + 1;
            int64_t dband = d / 2, drand = d - dband;
            if (dband > bhi - blo) dband = bhi - blo, drand = d - dband;
            distinct_in_range(&g, blo, bhi, dband, NULL, 0, c);
            if (!excl) excl = (int32_t *)malloc(sizeof(int32_t) * (size_t)(d + 1));
            else excl = (int32_t *)realloc(excl, sizeof(int32_t) * (size_t)(d + 1));
            memcpy(excl, c, sizeof(int32_t) * (size_t)dband);
            distinct_in_range(&g, 0, J->n, drand, excl, dband, c + dband);
            qsort(c, (size_t)d, sizeof(int32_t), cmp_i32);
        }
        rng_t gv = rng_for(J->seed, PURPOSE_VALS, (uint64_t)r);
        double *v = J->val + p0;
        for (int64_t i = 0; i < d; i++) {
            if (J->val_kind == VAL_NORMAL) v[i] = rng_normal(&gv);
            else if (J->val_kind == VAL_U01) v[i] = rng_u01(&gv);
            else v[i] = 2.0 * rng_u01(&gv) - 1.0;
        }
    }
    free(excl);
}

static void *fill_thread(void *arg) {
    fill_job *J = (fill_job *)arg;
    fill_rows(J, J->chunk_lo, J->chunk_hi);
    return NULL;
}

/* Fill columns/values of rows [r0, r1) given the global row pointer.
 * col/val point at the storage of row r0 (offset row_ptr[r0]). */
int wl_fill_rows(int kind, int val_kind, int64_t m, int64_t n, int64_t band,
                 uint64_t seed, int64_t r0, int64_t r1, const int64_t *row_ptr,
                 int32_t *col, double *val, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    fill_job base;
    memset(&base, 0, sizeof(base));
    base.kind = kind; base.val_kind = val_kind; base.m = m; base.n = n;
    base.r0 = r0; base.r1 = r1; base.band = band; base.seed = seed;
    base.row_ptr = row_ptr; base.base = row_ptr[r0]; base.col = col; base.val = val;
    fill_job jobs[256];
    pthread_t th[256];
    /* chunk by nnz so long rows are spread over threads */
    int64_t total = row_ptr[r1] - row_ptr[r0];
    int64_t r = r0;
    int used = 0;
    for (int t = 0; t < nthreads && r < r1; t++) {
        int64_t target = row_ptr[r0] + (total * (t + 1)) / nthreads;
        int64_t e = r;
        while (e < r1 && (row_ptr[e + 1] <= target || e == r)) e++;
        if (t == nthreads - 1) e = r1;
        jobs[t] = base;
        jobs[t].chunk_lo = r;
        jobs[t].chunk_hi = e;
        r = e;
        used = t + 1;
    }
    for (int t = 0; t < used; t++) pthread_create(&th[t], NULL, fill_thread, &jobs[t]);
    for (int t = 0; t < used; t++) pthread_join(th[t], NULL);
    return 0;
}
