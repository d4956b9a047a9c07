/* svdsc_paper.h -- the paper's own C interface of svds-C, on top of libsvdsc.
 *
 * PAPER.md:289-317 (Section 2.3, "Interface of svds-C"):
 *   svds_C(A, U, S, V, k)               svds_C_opt(A, U, S, V, k, tol, t, r)
 *   svds_C_dense(A, U, S, V, k)         svds_C_dense_opt(A, U, S, V, k, tol, t, r)
 * A sparse input uses the MKL four-array CSR layout of the paper (mat_csr):
 * 1-based column indices `cols` and per-row `pointerB` / `pointerE`, where
 * cols[pointerB[i]-1 .. pointerE[i]-2] are row i's entries (pointerE is
 * exclusive: reading Q13 of DESIGN.md).  Dense inputs and all
 * outputs use `mat`: nrows x ncols, column-major `d`.  Outputs U (nrows x k),
 * S (k x 1) and V (ncols x k) are allocated by the library with malloc
 * ("mallocated automatically in svds_C"); release them with
 * svdsc_mat_free.  All buffers here are HOST memory: the call copies A to the
 * current CUDA device, runs svdsc_solve there and copies the results back.
 *
 * Defaults of svds_C / svds_C_dense:
 *   tol = 1e-10, t = max(15, 3k) (clamped to min(m, n) - 1), r = 10 restarts.
 * `r` is the maximum number of augmented-restart passes (reading Q5).
 *
 * Return value: svdsc_status (include/svdsc.h); SVDSC_NOT_CONVERGED (1) means
 * the outputs are valid but some residual is >= tol after r passes.
 * Thread safety: each call uses its own library handle; distinct calls may run
 * concurrently on distinct threads.
 */
#ifndef SVDSC_PAPER_H
#define SVDSC_PAPER_H

#include <stdint.h>

#include "svdsc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* the paper's mat_csr (MKL LP64 four-array CSR, 1-based) */
typedef struct {
    int64_t nnz, nrows, ncols;
    double *values;   /* nnz */
    int *cols;        /* nnz, 1-based column indices */
    int *pointerB;    /* nrows, 1-based start of row i in cols/values */
    int *pointerE;    /* nrows, 1-based one-past-the-end of row i */
} svdsc_mat_csr;

/* the paper's mat: column-major nrows x ncols */
typedef struct {
    int64_t nrows, ncols;
    double *d;
} svdsc_mat;

SVDSC_API svdsc_status svds_C(const svdsc_mat_csr *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k);
SVDSC_API svdsc_status svds_C_opt(const svdsc_mat_csr *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k,
                                  double tol, int t, int r);
SVDSC_API svdsc_status svds_C_dense(const svdsc_mat *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k);
SVDSC_API svdsc_status svds_C_dense_opt(const svdsc_mat *A, svdsc_mat *U, svdsc_mat *S, svdsc_mat *V, int k,
                                        double tol, int t, int r);

/* free a mat allocated by this library (d set to NULL; NULL-safe) */
SVDSC_API void svdsc_mat_free(svdsc_mat *M);
SVDSC_API void svdsc_mat_csr_free(svdsc_mat_csr *A);

/* The paper layout -> the canonical 0-based CSR of svdsc_matrix_csr (host):
 * row_ptr[nrows+1], col_idx[nnz_kept], values[nnz_kept]; gaps between
 * pointerE[i] and pointerB[i+1] (legal in the four-array layout) are dropped
 * (SPEC.md:421).  Outputs are malloc'ed (free with free()).  EINVAL on
 * pointerE[i] < pointerB[i], pointers outside 1..nnz+1 or columns outside
 * 1..ncols (svdsc_paper_last_error names the row). */
SVDSC_API svdsc_status svdsc_paper_csr_to_csr(const svdsc_mat_csr *A, int64_t **row_ptr, int32_t **col_idx,
                                              double **values, int64_t *nnz_kept);

/* Matrix Market reader (host).  `coordinate real|integer general|symmetric`
 * -> *A in the paper layout (rows sorted by column, duplicates summed,
 * symmetric files expanded to both triangles), *is_dense = 0; `array real
 * general` -> *D (column-major), *is_dense = 1.  EINVAL with a line number in
 * svdsc_paper_last_error on malformed input. */
SVDSC_API svdsc_status svdsc_read_mm(const char *path, svdsc_mat_csr *A, svdsc_mat *D, int *is_dense);
/* Matrix Market writer: coordinate (general) for A, or array for D (exactly
 * one non-NULL); 17 significant digits (lossless round trip). */
SVDSC_API svdsc_status svdsc_write_mm(const char *path, const svdsc_mat_csr *A, const svdsc_mat *D);

/* message of the last failing call of this file's functions on this thread */
SVDSC_API const char *svdsc_paper_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SVDSC_PAPER_H */
