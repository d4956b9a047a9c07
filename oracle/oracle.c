/*
 * oracle.c -- plain, slow, single-threaded fp64 CPU oracle of svds-C.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2405_18966_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes: the restarted truncated SVD of arXiv 2405.18966
 * ("svds-C"), written step by step in the paper's order and notation:
 *   - Alg. 1 (Lanczos bidiagonalization) with the full
 *     re-orthogonalization of PAPER.md:121, done as two classical
 *     Gram-Schmidt passes (reading Q1 in DESIGN.md),
 *   - Proposition 1 / Eq. (4) residuals,
 *   - the augmented restart of Eqs. (5)-(7) / Alg. 2 steps 8-12
 *     (PAPER.md:147-184),
 *   - Alg. 2 final assembly, steps 15-16.
 * The small SVD of T (Alg. 2 step 4; the paper calls
 * LAPACKE_dgesvd) is a one-sided (Hestenes) Jacobi SVD with
 * cyclic-by-rows ordering, as the SPEC's dense_svd module suggests
 * (SPEC.md:141-159).
 *
 * Style rules (so a reader can check it against the paper by eye):
 *   no BLAS, no threads, no blocking, no fusion; every reduction is a plain
 *   left-to-right loop.  Compiled with -O2 -ffp-contract=off (no FMA).
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"): SPEC hand examples,
 * numpy.linalg.svd on random small matrices, closed-form spectra (Decay2,
 * sigma_i = exp(-i/40)), diagonal / U diag V^T matrices, the exact LBP
 * invariants, Eq. (6) identity after restart, matvec counts of Eq. (8).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_NOT_CONVERGED 1
#define OR_EINVAL -1
#define OR_ENOMEM -2
#define OR_ESVD_NOCONV -5
#define OR_ERANKDEF -6

/* ------------------------------------------------------------------ */
/* Matrix operand: CSR (0-based) or column-major dense     */
/* (the paper's `mat`).                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int kind; /* 0 = CSR, 1 = dense column-major */
    int64_t m, n;
    const int64_t *row_ptr; /* m+1 */
    const int32_t *col_idx; /* nnz */
    const double *val;      /* nnz */
    const double *dense;    /* m x n, leading dimension ld */
    int64_t ld;
} or_matrix;

/* y = A x  (Alg. 1 line 2 / line 7; MKL_dcsrmv PAPER.md:267) */
void or_spmv(int64_t m, const int64_t *row_ptr, const int32_t *col_idx,
             const double *val, const double *x, double *y) {
    for (int64_t r = 0; r < m; r++) {
        double s = 0.0;
        for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++)
            s += val[p] * x[col_idx[p]];
        y[r] = s;
    }
}

/* y = A^T x without materializing A^T (Alg. 1 line 5).
 * Each y[c] accumulates in increasing row order. */
void or_spmv_t(int64_t m, int64_t n, const int64_t *row_ptr,
               const int32_t *col_idx, const double *val, const double *x,
               double *y) {
    for (int64_t c = 0; c < n; c++) y[c] = 0.0;
    for (int64_t r = 0; r < m; r++)
        for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; p++)
            y[col_idx[p]] += val[p] * x[r];
}

/* y = A x, A column-major m x n with leading dimension ld (svds_C_dense,
 * PAPER.md:315-317).  Row r sums over columns in increasing order. */
void or_gemv_n(int64_t m, int64_t n, const double *A, int64_t ld,
               const double *x, double *y) {
    for (int64_t r = 0; r < m; r++) {
        double s = 0.0;
        for (int64_t c = 0; c < n; c++) s += A[r + c * ld] * x[c];
        y[r] = s;
    }
}

/* y = A^T x, A column-major. */
void or_gemv_t(int64_t m, int64_t n, const double *A, int64_t ld,
               const double *x, double *y) {
    for (int64_t c = 0; c < n; c++) {
        double s = 0.0;
        for (int64_t r = 0; r < m; r++) s += A[r + c * ld] * x[r];
        y[c] = s;
    }
}

static void mat_mul(const or_matrix *A, const double *x, double *y) {
    if (A->kind == 0)
        or_spmv(A->m, A->row_ptr, A->col_idx, A->val, x, y);
    else
        or_gemv_n(A->m, A->n, A->dense, A->ld, x, y);
}

static void mat_mul_t(const or_matrix *A, const double *x, double *y) {
    if (A->kind == 0)
        or_spmv_t(A->m, A->n, A->row_ptr, A->col_idx, A->val, x, y);
    else
        or_gemv_t(A->m, A->n, A->dense, A->ld, x, y);
}

/* ||x||_2 = sqrt(sum x_i^2), left to right (Alg. 1 lines 3, 6, 8). */
double or_norm2(int64_t len, const double *x) {
    double s = 0.0;
    for (int64_t i = 0; i < len; i++) s += x[i] * x[i];
    return sqrt(s);
}

/* Full re-orthogonalization: w <- (I - Q Q^T) w with
 * Q = first `ncols` columns of the column-major basis (leading dim ld).
 * Done twice (classical Gram-Schmidt, two passes; reading Q1):
 *   repeat 2x { h = Q^T w;  w = w - Q h }.
 * h is a caller scratch of length >= ncols. */
void or_cgs2(int64_t N, int64_t ncols, const double *Q, int64_t ld, double *w,
             double *h) {
    for (int pass = 0; pass < 2; pass++) {
        for (int64_t j = 0; j < ncols; j++) {
            double s = 0.0;
            for (int64_t r = 0; r < N; r++) s += Q[r + j * ld] * w[r];
            h[j] = s;
        }
        for (int64_t r = 0; r < N; r++) {
            double s = 0.0;
            for (int64_t j = 0; j < ncols; j++) s += Q[r + j * ld] * h[j];
            w[r] -= s;
        }
    }
}

/* Counter-based generator for breakdown replacement vectors (Q7):
 * element r of stream `stream` is uniform in [-1, 1), built from SplitMix64
 * of (seed, stream, r) using integer arithmetic only, so the CUDA side can
 * reproduce it bit for bit with its own implementation. */
static uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
double or_breakdown_uniform(uint64_t seed, uint64_t stream, uint64_t r) {
    uint64_t key = splitmix64(seed ^ splitmix64(stream * 0xD1B54A32D192ED03ULL + 1ULL));
    uint64_t z = splitmix64(key + r * 0x9E3779B97F4A7C15ULL);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

/* ------------------------------------------------------------------ */
/* One-sided Jacobi SVD of a p x q column-major matrix M (q <= p).     */
/* Alg. 2 step 4 small SVD.            */
/* Outputs: U (p x q, ld p), S (q, descending), V (q x q, ld q).       */
/* Returns number of sweeps used, or OR_ESVD_NOCONV.                   */
/* ------------------------------------------------------------------ */
int or_jacobi_svd(int64_t p, int64_t q, const double *M, double *U, double *S,
                  double *V, int max_sweeps) {
    double *W = (double *)malloc(sizeof(double) * (size_t)(p * q));
    double *Vw = (double *)malloc(sizeof(double) * (size_t)(q * q));
    double *Sw = (double *)malloc(sizeof(double) * (size_t)q);
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)q);
    if (!W || !Vw || !Sw || !perm) {
        free(W); free(Vw); free(Sw); free(perm);
        return OR_ENOMEM;
    }
    memcpy(W, M, sizeof(double) * (size_t)(p * q));
    for (int64_t j = 0; j < q; j++)
        for (int64_t i = 0; i < q; i++) Vw[i + j * q] = (i == j) ? 1.0 : 0.0;
    /* rotation threshold: |gamma| > 2 p eps sqrt(alpha*beta).  2 p eps bounds the
     * rounding error of a length-p dot product (gamma_p), so a pair that is
     * orthogonal to working precision is never rotated again and the sweep
     * loop terminates (reading Q10a). */
    const double ctol = 2.0 * (double)p * 2.220446049250313e-16;
    /* numerically zero columns (reading Q10b): a column whose norm is
     * <= p eps ||M||_F carries only rounding noise; it is never rotated and its
     * singular value is reported as exactly 0 (U completed orthonormally). */
    double normF = 0.0;
    for (int64_t i = 0; i < p * q; i++) normF += M[i] * M[i];
    const double tiny = (double)p * 2.220446049250313e-16 * sqrt(normF);
    int sweeps = 0, converged = 0;
    for (sweeps = 1; sweeps <= max_sweeps; sweeps++) {
        int rotated = 0;
        for (int64_t a = 0; a < q - 1; a++) {
            for (int64_t b = a + 1; b < q; b++) {
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (int64_t r = 0; r < p; r++) {
                    alpha += W[r + a * p] * W[r + a * p];
                    beta += W[r + b * p] * W[r + b * p];
                    gamma += W[r + a * p] * W[r + b * p];
                }
                if (!(sqrt(alpha) > tiny) || !(sqrt(beta) > tiny)) continue;
                if (fabs(gamma) <= ctol * sqrt(alpha) * sqrt(beta)) continue;
                rotated = 1;
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = (zeta >= 0.0 ? 1.0 : -1.0) /
                           (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = c * t;
                for (int64_t r = 0; r < p; r++) {
                    double wa = W[r + a * p], wb = W[r + b * p];
                    W[r + a * p] = c * wa - s * wb;
                    W[r + b * p] = s * wa + c * wb;
                }
                for (int64_t r = 0; r < q; r++) {
                    double va = Vw[r + a * q], vb = Vw[r + b * q];
                    Vw[r + a * q] = c * va - s * vb;
                    Vw[r + b * q] = s * va + c * vb;
                }
            }
        }
        if (!rotated) { converged = 1; break; }
    }
    if (!converged) {
        free(W); free(Vw); free(Sw); free(perm);
        return OR_ESVD_NOCONV;
    }
    for (int64_t j = 0; j < q; j++) {
        Sw[j] = or_norm2(p, W + j * p);
        if (!(Sw[j] > tiny)) Sw[j] = 0.0;
        perm[j] = j;
    }
    /* stable descending sort of the singular values (ties keep natural order) */
    for (int64_t i = 1; i < q; i++) {
        int64_t pj = perm[i];
        int64_t k = i - 1;
        while (k >= 0 && Sw[perm[k]] < Sw[pj]) { perm[k + 1] = perm[k]; k--; }
        perm[k + 1] = pj;
    }
    for (int64_t j = 0; j < q; j++) {
        int64_t src = perm[j];
        S[j] = Sw[src];
        for (int64_t r = 0; r < q; r++) V[r + j * q] = Vw[r + src * q];
        if (Sw[src] > 0.0) {
            for (int64_t r = 0; r < p; r++) U[r + j * p] = W[r + src * p] / Sw[src];
        } else {
            /* zero singular value: complete U with the standard basis vector
             * e_best whose component orthogonal to U(:,1:j) (two Gram-Schmidt
             * passes) is largest, normalized. */
            int64_t best = 0;
            double bestn = -1.0;
            for (int pick = 0; pick < 2; pick++) {
                for (int64_t e = (pick ? best : 0); e < (pick ? best + 1 : p); e++) {
                    for (int64_t r = 0; r < p; r++) U[r + j * p] = (r == e) ? 1.0 : 0.0;
                    for (int pass = 0; pass < 2; pass++)
                        for (int64_t jj = 0; jj < j; jj++) {
                            double d = 0.0;
                            for (int64_t r = 0; r < p; r++) d += U[r + jj * p] * U[r + j * p];
                            for (int64_t r = 0; r < p; r++) U[r + j * p] -= d * U[r + jj * p];
                        }
                    double nn = or_norm2(p, U + j * p);
                    if (!pick && nn > bestn) { bestn = nn; best = e; }
                    if (pick)
                        for (int64_t r = 0; r < p; r++) U[r + j * p] /= nn;
                }
            }
        }
        /* sign rule: largest-|.| entry of u_j made >= 0,
         * first index on ties; v_j flips with it. */
        int64_t imax = 0;
        double amax = -1.0;
        for (int64_t r = 0; r < p; r++)
            if (fabs(U[r + j * p]) > amax) { amax = fabs(U[r + j * p]); imax = r; }
        if (U[imax + j * p] < 0.0) {
            for (int64_t r = 0; r < p; r++) U[r + j * p] = -U[r + j * p];
            for (int64_t r = 0; r < q; r++) V[r + j * q] = -V[r + j * q];
        }
    }
    free(W); free(Vw); free(Sw); free(perm);
    return sweeps;
}

/* ------------------------------------------------------------------ */
/* Restarted truncated SVD: Alg. 2 with LBP =       */
/* Alg. 1 + full re-orthogonalization.               */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t k;          /* rank parameter */
    double tol;         /* relative residual tolerance (Eq. 4) */
    int32_t t;          /* subspace dimension; <= 0 -> max(15, 3k) (Alg. 2 step 1) */
    int32_t maxit;      /* r: maximum number of passes (Q5) */
    int32_t fixed_passes; /* >0: run exactly this many passes (parity hook, Q18) */
    int32_t reorth;     /* 2 = CGS2 (default), 1 = partial (PRO, reading Q20),
                           0 = off (test-only) */
    uint64_t seed;      /* breakdown-vector stream seed */
    double pro_delta;   /* PRO threshold; <= 0 -> sqrt(eps) (reading Q20) */
} or_opts;

typedef struct {
    int32_t passes, restarts, converged, t_used;
    int64_t steps, matvecs, breakdowns;
    double max_resid;
    int64_t reorths;   /* Lanczos half-steps whose vector was re-orthogonalized */
} or_info;

typedef struct {
    const or_matrix *A;
    const or_opts *o;
    double *U, *V, *T; /* U: m x (t+1), V: n x (t+1), T: (t+1) x (t+1) col-major */
    int64_t t;
    double amax;       /* largest |alpha|, |beta| seen so far (Q7) */
    uint64_t bd_stream;
    or_info *info;
    double *h;         /* scratch for CGS2 */
    /* PRO (reorth = 1): mu[l] ~ u_newest^T u_l, nu[l] ~ v_newest^T v_l */
    double *mu, *nu, *tmp;
    int force_u, force_v;
} or_state;

#define Tm(S, i, j) ((S)->T[(i) + (j) * ((S)->t + 1)]) /* 0-based */

static void reorth(or_state *S, int64_t N, int64_t ncols, const double *Q,
                   double *w) {
    if (S->o->reorth == 0 || ncols == 0) return;
    or_cgs2(N, ncols, Q, N, w, S->h);
}

/* Normalize w (length N) into `out` after the breakdown rule (Q7): if
 * ||w|| <= 1e-14 * max(amax, 1), replace w by a fresh counter-RNG vector,
 * re-orthogonalize it against Q(:, 1:ncols), set the T entry to 0.
 * Returns the value stored in T. */
static double finish_vector(or_state *S, int64_t N, int64_t ncols,
                            const double *Q, double *w, double *out) {
    double nrm = or_norm2(N, w);
    double thr = 1e-14 * (S->amax > 1.0 ? S->amax : 1.0);
    double tval = nrm;
    if (!(nrm > thr)) {
        tval = 0.0;
        S->info->breakdowns++;
        uint64_t stream = S->bd_stream++;
        for (int64_t r = 0; r < N; r++)
            w[r] = or_breakdown_uniform(S->o->seed, stream, (uint64_t)r);
        if (ncols > 0) or_cgs2(N, ncols, Q, N, w, S->h);
        nrm = or_norm2(N, w);
    } else if (nrm > S->amax) {
        S->amax = nrm;
    }
    for (int64_t r = 0; r < N; r++) out[r] = w[r] / nrm;
    return tval;
}

/* ------------------------------------------------------------------ */
/* Partial re-orthogonalization (reorth = 1; reading  */
/* Q20 of DESIGN.md).  The paper names this class -- PROPACK lansvd,   */
/* "Lanczos bidiagonalization process with partial re-orthogonalization"*/
/* -- without giving its rules; this is the omega        */
/* recurrence of Simon (Lanczos) as extended by Larsen to the          */
/* bidiagonalization, restated for the T of this algorithm (first pass:*/
/* upper bidiagonal; after a restart: the arrow of Alg. 2 step 9).     */
/*                                                                     */
/* With 0-based columns, T holds the relations                         */
/*   A v_l   = sum_{p<=l} T(p,l) u_p   (column l of T)                  */
/*   A^T u_l = sum_{p>=l} T(l,p) v_p   (row l of T)                     */
/* (Alg. 1 lines 5-8; Eqs. (5)-(7) after a restart).  If mu[p] are the   */
/* inner products of u_{i-1} with u_p and nu[l] those of v_{i-1} with   */
/* v_l, then v_i = (A^T u_{i-1} - alpha v_{i-1}) / beta has             */
/*   beta * (v_i^T v_l) = sum_{p<=l} T(p,l) mu[p] - alpha * nu[l],      */
/* and u_i = (A v_i - beta u_{i-1}) / alpha has                         */
/*   alpha * (u_i^T u_l) = sum_{p>=l, p<=i} T(l,p) nu[p] - beta * mu[l] */
/* with nu now the row of v_i.  Rounding enters as a term of size      */
/* eps1 = eps * anorm with the sign of the sum (Simon's model), anorm  */
/* the largest column 1-norm of T seen so far.                          */
/* ------------------------------------------------------------------ */
#define OR_EPS 2.220446049250313e-16 /* 2^-52 */

/* largest column 1-norm of T(:, 0:ncols-1) */
double or_pro_anorm(const double *T, int64_t ldt, int64_t ncols) {
    double a = 0.0;
    for (int64_t l = 0; l < ncols; l++) {
        double c = 0.0;
        for (int64_t p = 0; p <= l; p++) c += fabs(T[p + l * ldt]);
        if (c > a) a = c;
    }
    return a;
}

/* nu (length i+1, in place): row of v_{i-1} -> row of v_i.  mu: row of
 * u_{i-1}.  alpha = T(i-1,i-1); beta = ||A^T u_{i-1} - alpha v_{i-1}||. */
void or_pro_nu_update(const double *T, int64_t ldt, int64_t i, const double *mu,
                      double *nu, double beta, double eps1) {
    double alpha = T[(i - 1) + (i - 1) * ldt];
    for (int64_t l = 0; l < i; l++) {
        double x = 0.0;
        for (int64_t p = 0; p <= l; p++) x += T[p + l * ldt] * mu[p];
        x -= alpha * nu[l];
        x += (x < 0.0) ? -eps1 : eps1;
        nu[l] = x / beta;
    }
    nu[i] = 1.0;
}

/* mu (length i+1, in place): row of u_{i-1} -> row of u_i.  nu: row of
 * v_i (nu[i] = 1).  beta = T(i-1,i); alpha = ||A v_i - beta u_{i-1}||. */
void or_pro_mu_update(const double *T, int64_t ldt, int64_t i, const double *nu,
                      double *mu, double alpha, double eps1) {
    double beta = T[(i - 1) + i * ldt];
    for (int64_t l = 0; l < i; l++) {
        double y = 0.0;
        for (int64_t p = l; p <= i; p++) y += T[l + p * ldt] * nu[p];
        y -= beta * mu[l];
        y += (y < 0.0) ? -eps1 : eps1;
        mu[l] = y / alpha;
    }
    mu[i] = 1.0;
}

/* The decision for the new vector x (length N, not yet normalized) whose
 * estimate row `row` (length i+1) was just updated: re-orthogonalize if
 * some |row[l]| exceeds delta, or if the previous vector of this side was
 * re-orthogonalized because of its estimate (*force; Larsen: the next
 * vector inherits the loss through the three-term relation).  A vector
 * that is re-orthogonalized has its row reset to eps. */
static int pro_decide(or_state *S, double *row, int64_t i, double nrm, int *force) {
    double delta = S->o->pro_delta > 0.0 ? S->o->pro_delta : sqrt(OR_EPS);
    int viol = !(nrm > 0.0);
    for (int64_t l = 0; l < i; l++)
        if (!(fabs(row[l]) <= delta)) viol = 1;
    int reo = viol || *force;
    *force = viol && !*force;
    if (reo) {
        for (int64_t l = 0; l < i; l++) row[l] = OR_EPS;
        S->info->reorths++;
    }
    return reo;
}

/* V side of step i (computing v_i from w): returns 1 -> re-orthogonalize */
static int pro_v(or_state *S, int64_t i, const double *w) {
    int64_t n = S->A->n, ldt = S->t + 1;
    double beta = or_norm2(n, w);
    double eps1 = OR_EPS * or_pro_anorm(S->T, ldt, i);
    or_pro_nu_update(S->T, ldt, i, S->mu, S->nu, beta, eps1);
    return pro_decide(S, S->nu, i, beta, &S->force_v);
}

/* U side of step i (computing u_i from z) */
static int pro_u(or_state *S, int64_t i, const double *z) {
    int64_t m = S->A->m, ldt = S->t + 1;
    double alpha = or_norm2(m, z);
    double eps1 = OR_EPS * or_pro_anorm(S->T, ldt, i);
    or_pro_mu_update(S->T, ldt, i, S->nu, S->mu, alpha, eps1);
    return pro_decide(S, S->mu, i, alpha, &S->force_u);
}

/* After the restart (Alg. 2 steps 8-11): V(:,0:k-1) = V(:,0:t-1) Vh(:,0:k-1)
 * and v_k = old v_t, so v_k^T v~_j = sum_l (v_t^T v_l) Vh(l,j); u_k was
 * re-orthogonalized in full, so its row is eps.  nu / mu:
 * length >= t+1 (in place), Vh: t x t column-major, tmp: k doubles. */
void or_pro_restart(int64_t t, int64_t k, const double *Vh, double *nu, double *mu, double *tmp) {
    for (int64_t j = 0; j < k; j++) {
        double s = 0.0;
        for (int64_t l = 0; l < t; l++) s += nu[l] * Vh[l + j * t];
        tmp[j] = s;
    }
    for (int64_t j = 0; j < k; j++) nu[j] = tmp[j];
    nu[k] = 1.0;
    for (int64_t j = 0; j < k; j++) mu[j] = OR_EPS;
    mu[k] = 1.0;
}

static void pro_restart(or_state *S, int64_t k, const double *Vh) {
    or_pro_restart(S->t, k, Vh, S->nu, S->mu, S->tmp);
    S->force_u = S->force_v = 0;
}

/* Alg. 1 loop body for i = i0..t (1-based), continuing from stored
 * U(:,1:i0), V(:,1:i0), T.  Computes v_{i+1}, beta_i, u_{i+1}, alpha_{i+1}.
 * The literal LBP(A, t+1) also forms u_{t+1} (Q2). */
static void lbp_steps(or_state *S, int64_t i0, double *w, double *z) {
    const or_matrix *A = S->A;
    int64_t m = A->m, n = A->n, t = S->t;
    for (int64_t i = i0; i <= t; i++) {
        /* line 5: v_{i+1} = A^T u_i - alpha_i v_i */
        double alpha_i = Tm(S, i - 1, i - 1);
        mat_mul_t(A, S->U + (i - 1) * m, w);
        S->info->matvecs++;
        for (int64_t r = 0; r < n; r++) w[r] -= alpha_i * S->V[r + (i - 1) * n];
        /* full re-orthogonalization against V^{(i)}; reorth = 1:
         * only when the omega estimate asks for it (reading Q20) */
        if (S->o->reorth == 1) {
            if (pro_v(S, i, w)) or_cgs2(n, i, S->V, n, w, S->h);
        } else {
            reorth(S, n, i, S->V, w);
            if (S->o->reorth == 2) S->info->reorths++;
        }
        /* line 6: beta_i = ||v_{i+1}||, v_{i+1} /= beta_i */
        double beta_i = finish_vector(S, n, i, S->V, w, S->V + i * n);
        Tm(S, i - 1, i) = beta_i;
        /* line 7: u_{i+1} = A v_{i+1} - beta_i u_i */
        mat_mul(A, S->V + i * n, z);
        S->info->matvecs++;
        for (int64_t r = 0; r < m; r++) z[r] -= beta_i * S->U[r + (i - 1) * m];
        if (S->o->reorth == 1) {
            if (pro_u(S, i, z)) or_cgs2(m, i, S->U, m, z, S->h);
        } else {
            reorth(S, m, i, S->U, z);
            if (S->o->reorth == 2) S->info->reorths++;
        }
        /* line 8: alpha_{i+1} = ||u_{i+1}||, u_{i+1} /= alpha_{i+1} */
        double alpha_ip1 = finish_vector(S, m, i, S->U, z, S->U + i * m);
        Tm(S, i, i) = alpha_ip1;
        S->info->steps++;
    }
}

/* Alg. 2.  v0 (length n) is the start vector before normalization
 * (Alg. 1 line 1, "randn(n,1)": supplied by the harness, reading Q8).
 * Outputs: S_out[k], U_out (m x k, ld m), V_out (n x k, ld n), resid[k]. */
int or_svds(const or_matrix *A, const or_opts *o, const double *v0,
            double *S_out, double *U_out, double *V_out, double *resid,
            or_info *info) {
    memset(info, 0, sizeof(*info));
    int64_t m = A->m, n = A->n, k = o->k;
    int64_t mn = m < n ? m : n;
    if (k < 1 || !(o->tol > 0.0) || m < 1 || n < 1) return OR_EINVAL;
    int64_t t = o->t > 0 ? o->t : (3 * k > 15 ? 3 * k : 15); /* Alg. 2 step 1 */
    if (t > mn - 1) t = mn - 1;                              /* clamp, Q14 */
    if (t < k + 2) return OR_EINVAL;
    int64_t maxit = o->maxit > 0 ? o->maxit : 10;
    info->t_used = (int32_t)t;

    or_state S;
    memset(&S, 0, sizeof(S));
    S.A = A; S.o = o; S.t = t; S.info = info;
    S.U = (double *)calloc((size_t)(m * (t + 1)), sizeof(double));
    S.V = (double *)calloc((size_t)(n * (t + 1)), sizeof(double));
    S.T = (double *)calloc((size_t)((t + 1) * (t + 1)), sizeof(double));
    S.h = (double *)calloc((size_t)(t + 2), sizeof(double));
    S.mu = (double *)calloc((size_t)(t + 2), sizeof(double));
    S.nu = (double *)calloc((size_t)(t + 2), sizeof(double));
    S.tmp = (double *)calloc((size_t)(t + 2), sizeof(double));
    double *w = (double *)calloc((size_t)n, sizeof(double));
    double *z = (double *)calloc((size_t)m, sizeof(double));
    double *Tt = (double *)calloc((size_t)(t * t), sizeof(double));
    double *Uh = (double *)calloc((size_t)(t * t), sizeof(double));
    double *Vh = (double *)calloc((size_t)(t * t), sizeof(double));
    double *Sh = (double *)calloc((size_t)t, sizeof(double));
    double *Uk = (double *)calloc((size_t)(m * k), sizeof(double));
    double *Vk = (double *)calloc((size_t)(n * k), sizeof(double));
    double *rho = (double *)calloc((size_t)k, sizeof(double));
    int status = OR_OK;
    if (!S.U || !S.V || !S.T || !S.h || !S.mu || !S.nu || !S.tmp || !w || !z || !Tt ||
        !Uh || !Vh || !Sh || !Uk || !Vk || !rho) {
        status = OR_ENOMEM;
        goto done;
    }

    /* Alg. 1 line 1: v_1 = v0 / ||v0|| */
    {
        double nv = or_norm2(n, v0);
        if (!(nv > 0.0)) { status = OR_EINVAL; goto done; }
        for (int64_t r = 0; r < n; r++) S.V[r] = v0[r] / nv;
    }
    /* lines 2-3: u_1 = A v_1, alpha_1 = ||u_1||, u_1 /= alpha_1 */
    mat_mul(A, S.V, z);
    info->matvecs++;
    Tm(&S, 0, 0) = finish_vector(&S, m, 0, S.U, z, S.U);
    S.mu[0] = 1.0; /* PRO rows of u_0, v_0 */
    S.nu[0] = 1.0;

    int64_t i0 = 1;
    int converged = 0;
    for (;;) {
        /* Alg. 2 step 2 / step 12: LBP from iteration i0 up to t (t+1 vectors) */
        lbp_steps(&S, i0, w, z);
        info->passes++;
        /* step 4: [Uh, Sh, Vh] = svd(T(1:t, 1:t)) */
        for (int64_t j = 0; j < t; j++)
            for (int64_t i = 0; i < t; i++) Tt[i + j * t] = Tm(&S, i, j);
        int sw = or_jacobi_svd(t, t, Tt, Uh, Sh, Vh, 50);
        if (sw < 0) { status = OR_ESVD_NOCONV; goto done; }
        /* step 5, Eq. (4): res_j = |T(t,t+1) Uh(t,j)| / Sh(j,j) */
        double beta_t = Tm(&S, t - 1, t);
        converged = 1;
        info->max_resid = 0.0;
        for (int64_t j = 0; j < k; j++) {
            double num = fabs(beta_t * Uh[(t - 1) + j * t]);
            double r;
            if (Sh[j] > 0.0) r = num / Sh[j];
            else if (num <= 1e-14) r = 0.0; /* SPEC.md:312 rank-deficient rule */
            else { status = OR_ERANKDEF; goto done; }
            resid[j] = r;
            if (!(r < o->tol)) converged = 0; /* strict '<' */
            if (r > info->max_resid) info->max_resid = r;
        }
        int stop;
        if (o->fixed_passes > 0) stop = (info->passes >= o->fixed_passes);
        else stop = converged || (info->passes >= maxit);
        if (stop) break;

        /* Augmented restart, Alg. 2 steps 8-12. */
        /* step 8: Uk = U(:,1:t) Uh(:,1:k), Vk = V(:,1:t) Vh(:,1:k) */
        for (int64_t j = 0; j < k; j++) {
            for (int64_t r = 0; r < m; r++) {
                double s = 0.0;
                for (int64_t l = 0; l < t; l++) s += S.U[r + l * m] * Uh[l + j * t];
                Uk[r + j * m] = s;
            }
            for (int64_t r = 0; r < n; r++) {
                double s = 0.0;
                for (int64_t l = 0; l < t; l++) s += S.V[r + l * n] * Vh[l + j * t];
                Vk[r + j * n] = s;
            }
        }
        /* step 9: beta_t = T(t,t+1); T = zeros(t+1);
         *         T(1:k,1:k+1) = [Sh(1:k,1:k), (beta_t Uh(t,1:k))^T] */
        for (int64_t j = 0; j < k; j++) rho[j] = beta_t * Uh[(t - 1) + j * t];
        memset(S.T, 0, sizeof(double) * (size_t)((t + 1) * (t + 1)));
        for (int64_t j = 0; j < k; j++) {
            Tm(&S, j, j) = Sh[j];
            Tm(&S, j, k) = rho[j];
        }
        /* step 10: v_{k+1} = v_{t+1} (listing typo P:237 read as v_{t+1}, Q3);
         *          u_{k+1} = A v_{k+1} - Uk rho   (Eq. 7) */
        memmove(S.V + k * n, S.V + t * n, sizeof(double) * (size_t)n);
        memcpy(S.U, Uk, sizeof(double) * (size_t)(m * k));
        memcpy(S.V, Vk, sizeof(double) * (size_t)(n * k));
        mat_mul(A, S.V + k * n, z);
        info->matvecs++;
        for (int64_t r = 0; r < m; r++) {
            double s = 0.0;
            for (int64_t j = 0; j < k; j++) s += S.U[r + j * m] * rho[j];
            z[r] -= s;
        }
        /* re-orthogonalization at step 10 */
        reorth(&S, m, k, S.U, z);
        /* step 11: alpha_{k+1} = ||u_{k+1}||, u_{k+1} /= alpha_{k+1} */
        Tm(&S, k, k) = finish_vector(&S, m, k, S.U, z, S.U + k * m);
        if (o->reorth == 1) pro_restart(&S, k, Vh);
        info->restarts++;
        i0 = k + 1; /* step 12 */
    }

    /* steps 15-16: S = diag(Sh(1:k)), U = U(:,1:t) Uh(:,1:k), V likewise */
    for (int64_t j = 0; j < k; j++) {
        S_out[j] = Sh[j];
        for (int64_t r = 0; r < m; r++) {
            double s = 0.0;
            for (int64_t l = 0; l < t; l++) s += S.U[r + l * m] * Uh[l + j * t];
            U_out[r + j * m] = s;
        }
        for (int64_t r = 0; r < n; r++) {
            double s = 0.0;
            for (int64_t l = 0; l < t; l++) s += S.V[r + l * n] * Vh[l + j * t];
            V_out[r + j * n] = s;
        }
    }
    info->converged = converged;
    if (status == OR_OK && !converged) status = OR_NOT_CONVERGED;

done:
    free(S.U); free(S.V); free(S.T); free(S.h); free(S.mu); free(S.nu); free(S.tmp);
    free(w); free(z); free(Tt);
    free(Uh); free(Vh); free(Sh); free(Uk); free(Vk); free(rho);
    return status;
}

/* Alg. 1 alone: LBP(A, t+1) from v0 (first pass, no restart).  Outputs the
 * bases U (m x (t+1)), V (n x (t+1)) and T ((t+1) x (t+1)), all column-major.
 * Used by the step-parity tests (alpha/beta sequences, orthogonality). */
int or_lbp(const or_matrix *A, const or_opts *o, int64_t t, const double *v0,
           double *U, double *V, double *T, or_info *info) {
    memset(info, 0, sizeof(*info));
    int64_t m = A->m, n = A->n;
    if (t < 1 || t + 1 > (m < n ? m : n)) return OR_EINVAL;
    or_state S;
    memset(&S, 0, sizeof(S));
    S.A = A; S.o = o; S.t = t; S.info = info;
    S.U = U; S.V = V; S.T = T;
    memset(U, 0, sizeof(double) * (size_t)(m * (t + 1)));
    memset(V, 0, sizeof(double) * (size_t)(n * (t + 1)));
    memset(T, 0, sizeof(double) * (size_t)((t + 1) * (t + 1)));
    S.h = (double *)calloc((size_t)(t + 2), sizeof(double));
    S.mu = (double *)calloc((size_t)(t + 2), sizeof(double));
    S.nu = (double *)calloc((size_t)(t + 2), sizeof(double));
    double *w = (double *)calloc((size_t)n, sizeof(double));
    double *z = (double *)calloc((size_t)m, sizeof(double));
    if (!S.h || !S.mu || !S.nu || !w || !z) {
        free(S.h); free(S.mu); free(S.nu); free(w); free(z);
        return OR_ENOMEM;
    }
    double nv = or_norm2(n, v0);
    for (int64_t r = 0; r < n; r++) V[r] = v0[r] / nv;
    mat_mul(A, V, z);
    info->matvecs++;
    Tm(&S, 0, 0) = finish_vector(&S, m, 0, U, z, U);
    S.mu[0] = 1.0;
    S.nu[0] = 1.0;
    lbp_steps(&S, 1, w, z);
    info->passes = 1;
    info->t_used = (int32_t)t;
    free(S.h); free(S.mu); free(S.nu); free(w); free(z);
    return OR_OK;
}
