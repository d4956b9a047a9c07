/*
 * svdsc.h -- C ABI of the B200-native svds-C hot path (libsvdsc.so).
 *
 * The library computes the k largest singular triplets of a sparse (CSR) or
 * dense fp64 matrix A (Eq. (1): A ~ U_k Sigma_k V_k^T) with the
 * augmented-restart Lanczos bidiagonalization of svds-C (Alg. 1 + full
 * re-orthogonalization; Alg. 2).  Every
 * step of the method runs in the library's own sm_100a kernels on the
 * caller's CUDA stream; there is no CPU fallback.
 *
 * Conventions (all entry points):
 *   - Pointers documented as "device" must be CUDA device pointers (e.g. torch
 *     CUDA tensors); "host" pointers are ordinary host memory.
 *   - Dense matrices and bases are column-major (the paper's `mat`,
 *     PAPER.md:298-302) with an explicit leading dimension >= nrows.
 *   - CSR matrices are 0-based: row_ptr[nrows+1] int64 (monotone, row_ptr[0]=0),
 *     col_idx[nnz] int32 in [0, ncols), values[nnz] fp64, finite.  Columns
 *     need not be sorted; duplicate (row, col) entries act as their sum
 *     (SPEC.md:112).  The paper's 1-based pointerB/pointerE layout
 *      is converted to this form by the caller
 *     (reading Q13).
 *   - Ownership: every input array stays owned by the caller and must stay
 *     valid and unmodified while a handle/matrix that references it lives.
 *     Outputs are caller-allocated (a departure from "mallocated
 *     automatically", so that the caller's allocator owns all
 *     device memory).  Objects created by the library are freed by the
 *     matching *_destroy call.
 *   - Errors: every function returns an svdsc_status.  Contract violations
 *     return SVDSC_EINVAL before any device work; a message is available from
 *     svdsc_last_error(handle).  CUDA/NCCL failures return SVDSC_ECUDA /
 *     SVDSC_ENCCL.  Functions are synchronous with respect to the host unless
 *     documented as "enqueued".
 *   - Threading: one call at a time per handle; distinct handles are
 *     independent.
 */
#ifndef SVDSC_H
#define SVDSC_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SVDSC_API __attribute__((visibility("default")))
#else
#define SVDSC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SVDSC_OK = 0,
    SVDSC_NOT_CONVERGED = 1,  /* results valid, some residual >= tol */
    SVDSC_EINVAL = -1,        /* contract violation; nothing was computed        */
    SVDSC_ENOMEM = -2,        /* device allocation failed                        */
    SVDSC_ECUDA = -3,         /* CUDA runtime error                               */
    SVDSC_ENCCL = -4,         /* NCCL error or NCCL library unavailable           */
    SVDSC_ESVD_NOCONV = -5,   /* small Jacobi SVD: no convergence in 50 sweeps    */
    SVDSC_ERANKDEF = -6       /* sigma_j = 0 with non-negligible residual */
} svdsc_status;

typedef struct svdsc_handle svdsc_handle;
typedef struct svdsc_matrix svdsc_matrix;

/* Options of Alg. 2 (defaults). */
typedef struct {
    int32_t k;            /* rank parameter, >= 1                                      */
    double tol;           /* relative residual tolerance of Eq. (4), > 0 (default 1e-10)*/
    int32_t t;            /* subspace dimension; <= 0 -> max(15, 3k) (Alg. 2 step 1),  */
                          /* clamped to min(m,n)-1; EINVAL if then t < k+2 (reading Q14)*/
    int32_t maxit;        /* r: maximum number of passes (reading Q5); <= 0 -> 10       */
    uint64_t seed;        /* seed of the internal start vector / breakdown streams      */
    const double *v0;     /* device, length ncols (global), or NULL -> internal N(0,1)  */
    int32_t fixed_passes; /* > 0: run exactly this many passes (parity hook, Q18)        */
    int32_t reorth;       /* 0 or 2 = CGS2 every half-step, the paper's method           */
                          /*     (0 so that a zero-initialized struct is   */
                          /*     the default);                                            */
                          /* 1 = partial: CGS2 only when the omega estimate of the loss  */
                          /*     of orthogonality exceeds sqrt(eps) (Q20;      */
                          /*     single GPU; PAPER.md:42 names the class);               */
                          /* -1 = off, test-only                           */
} svdsc_opts;

typedef struct {
    int32_t passes, restarts, converged, t_used;
    int64_t steps;        /* Lanczos steps (one A^T u and one A v product each)          */
    int64_t matvecs;      /* products with A or A^T actually performed                   */
    int64_t breakdowns;   /* breakdown replacements (reading Q7)                          */
    double max_resid;     /* max_j of Eq. (4) residuals at the final check               */
    double seconds_total; /* host wall time of svdsc_solve                                */
    int64_t launches;     /* kernels launched by the library during the solve            */
    int64_t bytes_model;  /* algorithmic HBM bytes of the Lanczos steps */
                          /* (with reorth = 1: as if every half-step re-orthogonalized)  */
    int64_t reorths;      /* Lanczos half-steps (A^T u or A v side) re-orthogonalized     */
    int64_t bytes_reorth; /* the CGS2 share of bytes_model: 8 N (3 i + 5) per           */
                          /* re-orthogonalization (+ 8 m k for the restart's U_k rho)    */
    double seconds_analysis; /* host wall time of the matrix's analysis (svdsc_matrix_*:  */
                          /* validation, row bins, CSC copy); the host-buffer entry      */
                          /* points include it in seconds_total                           */
} svdsc_info;

/* ---- handles --------------------------------------------------------------- */
/* Create a handle bound to the current CUDA device and `stream` (a cudaStream_t;
 * NULL = legacy default stream).  Owns internal scratch (device). */
SVDSC_API svdsc_status svdsc_create(svdsc_handle **h, void *stream);
SVDSC_API svdsc_status svdsc_set_stream(svdsc_handle *h, void *stream);
SVDSC_API void svdsc_destroy(svdsc_handle *h);
/* Last error message of this handle (static storage owned by the handle). */
SVDSC_API const char *svdsc_last_error(const svdsc_handle *h);
/* Library version string, e.g. "svdsc 0.1 sm_100a". */
SVDSC_API const char *svdsc_version(void);

/* ---- matrices ---------------------------------------------------------------
 * Analysis (once per matrix, "mallocate ... at the beginning"):
 * validation, row-length binning, and a device-built CSC copy used for A^T u.
 * For a row-partitioned multi-GPU run each rank passes its local rows
 * [row_offset, row_offset + nrows) of the m_global x ncols matrix with global
 * column indices.  Single GPU: row_offset = 0,
 * m_global = nrows.  Device arrays: row_ptr, col_idx, values / data. */
SVDSC_API svdsc_status svdsc_matrix_csr(svdsc_handle *h, int64_t nrows, int64_t ncols, int64_t nnz,
                              const int64_t *row_ptr, const int32_t *col_idx,
                              const double *values, int64_t row_offset, int64_t m_global,
                              svdsc_matrix **M);
SVDSC_API svdsc_status svdsc_matrix_dense(svdsc_handle *h, int64_t nrows, int64_t ncols, int64_t ld,
                                const double *data, int64_t row_offset, int64_t m_global,
                                svdsc_matrix **M);
SVDSC_API void svdsc_matrix_destroy(svdsc_matrix *M);

/* ---- the solve (Alg. 2) -----------------------------------------------------
 * Device workspace bytes needed by svdsc_solve for these options. */
SVDSC_API svdsc_status svdsc_workspace_size(svdsc_matrix *M, const svdsc_opts *o, size_t *bytes);
/* Compute S[k] (descending), U (m_local x k, ld ldu >= m_local), V (ncols x k,
 * ld ldv >= ncols; replicated on every rank), resid[k] (Eq. (4) residuals).
 * S, U, V, resid are device pointers (resid may be NULL).  workspace: device,
 * >= svdsc_workspace_size bytes, or NULL (the library allocates and frees it).
 * info: host, may be NULL.  Returns after the results are complete on the
 * handle's stream.  SVDSC_NOT_CONVERGED still fills every output. */
SVDSC_API svdsc_status svdsc_solve(svdsc_matrix *M, const svdsc_opts *o, void *workspace,
                         size_t ws_bytes, double *S, double *U, int64_t ldu, double *V,
                         int64_t ldv, double *resid, svdsc_info *info);

/* End-to-end convenience with HOST buffers: copies A (and v0 if given) from
 * host memory, analyses, solves, copies S, U (m x k, ld m), V (n x k, ld n) and
 * resid back to host.  All pointers here are host pointers (pinned memory is
 * fastest); opts->v0, if non-NULL, is a HOST pointer of length n. */
SVDSC_API svdsc_status svdsc_solve_host_csr(svdsc_handle *h, int64_t m, int64_t n, int64_t nnz,
                                  const int64_t *row_ptr, const int32_t *col_idx,
                                  const double *values, const svdsc_opts *o, double *S,
                                  double *U, double *V, double *resid, svdsc_info *info);
SVDSC_API svdsc_status svdsc_solve_host_dense(svdsc_handle *h, int64_t m, int64_t n,
                                    const double *data /* col-major, ld m */,
                                    const svdsc_opts *o, double *S, double *U, double *V,
                                    double *resid, svdsc_info *info);

/* ---- step-level entry points (the hot-path rows of SURVEY.md 8(a)) -------- */
/* a1 / a5: y = op(A) x - c * yprev, op = A (trans=0, Alg. 1 line 7) or A^T
 * (trans=1, Alg. 1 line 5).  x, y, yprev device; c_dev is a device pointer to
 * the scalar c (may be NULL: c = 0, yprev ignored).  Enqueued on the stream. */
SVDSC_API svdsc_status svdsc_op_matvec(svdsc_matrix *M, int trans, const double *x, double *y,
                             const double *c_dev, const double *yprev);
/* a2-a4 / a6: one re-orthogonalization half-step of the solver: two-pass
 * classical Gram-Schmidt of w (length N, device, 16-byte aligned for the
 * streaming kernels) against the first ncols columns of the column-major basis
 * Q (ld >= N), then beta = ||w|| (Alg. 1 lines 6 / 8) and
 * w <- w / beta.  *norm_dev (device scalar, may be NULL) = beta; a breakdown
 * (beta <= 1e-14, reading Q7) gives beta = 0 and leaves w unnormalized.  The
 * kernel is the one the solver picks for this shape (svdsc_set_policy
 * SVDSC_POLICY_CGS2 overrides).  Synchronous. */
SVDSC_API svdsc_status svdsc_op_cgs2(svdsc_handle *h, int64_t N, int64_t ncols, const double *Q,
                           int64_t ldq, double *w, double *norm_dev);
/* a2-a4 / a6 across P row-partitioned ranks, the multi-GPU re-orthogonalization
 * of SURVEY.md 8(f2) (BASELINE.json north_star (e): all-reduce of the
 * Gram-Schmidt coefficient vectors): ONE kernel per half-step whose two global
 * reductions (h1 = Q^T w and [h2 = Q^T w'; ||w'||^2]) and the rare
 * explicit norm are completed across the ranks inside the kernel -- each rank
 * pushes its column sums into every rank's mailbox and sums the P slots in rank
 * order.  The solver runs this kernel for P > 1 over NCCL (one process per GPU,
 * mailboxes mapped through CUDA IPC / NVLink).  This entry point EMULATES P
 * ranks on the handle's one GPU as P groups of CTAs of one cooperative launch
 * (kernels that wait on one another are never separate launches on one GPU),
 * each group with its own operands, scratch and mailbox: the same kernel code
 * and protocol, for tests.
 *   P: 1..8 ranks; row0: host array of P+1 row offsets (row0[0] = 0,
 *   row0[P] = N, every row0[q] even, every rank >= 1 row); rank q owns rows
 *   [row0[q], row0[q+1]) of the device basis Q (N x ncols, column-major,
 *   ldq >= N, even, 16-byte aligned; ncols <= 384) and of the device vector w
 *   (16-byte aligned), re-orthogonalized and normalized in place.
 *   beta_out: host array of P: the norm each rank computed (bitwise equal on
 *   every rank; 0 on breakdown, reading Q7).
 * Errors: SVDSC_EINVAL (arguments), SVDSC_ECUDA (launch; e.g. fewer than P
 * SMs), SVDSC_ENCCL (a group never arrived: protocol failure).  Synchronous. */
SVDSC_API svdsc_status svdsc_op_cgs2_peer_emulate(svdsc_handle *h, int32_t P, const int64_t *row0,
                                                  int64_t ncols, const double *Q, int64_t ldq, double *w,
                                                  double *beta_out);
/* a7: SVD of the p x p column-major device matrix Tm (Alg. 2 step 4) by the
 * device one-sided Jacobi: U, V (p x p, ld p) and S (p, descending), sign rule
 * of SPEC.md:158.  Returns SVDSC_ESVD_NOCONV after 50 sweeps.  Synchronous. */
SVDSC_API svdsc_status svdsc_op_small_svd(svdsc_handle *h, int32_t p, const double *Tm, double *U,
                                double *S, double *V, int32_t *sweeps);
/* a8 / a9: Qout(:, 0:k) = Q(:, 0:t) W(:, 0:k) for N rows; Qout may equal Q (in
 * place, the restart's Ritz recombination, Alg. 2 step 8).  W is t x >=k
 * column-major device (ld ldw).  Enqueued. */
SVDSC_API svdsc_status svdsc_op_recombine(svdsc_handle *h, int64_t N, int32_t t, int32_t k,
                                const double *Q, int64_t ldq, const double *W, int32_t ldw,
                                double *Qout, int64_t ldo);
/* One first pass LBP(A, t+1) from v0 (device, length ncols): bases U
 * (m x (t+1), ld ldu), V (n x (t+1), ld ldv) and T ((t+1) x (t+1), col-major,
 * device).  The GPU path does not form u_{t+1} (reading Q2): column t of U
 * and T(t,t) are left zero.  Synchronous. */
SVDSC_API svdsc_status svdsc_op_lbp(svdsc_matrix *M, const svdsc_opts *o, int32_t t, const double *v0,
                          double *U, int64_t ldu, double *V, int64_t ldv, double *T,
                          svdsc_info *info);

/* ---- profiling ----------------------------------------------------------------
 * When enabled, svdsc_solve brackets each operation family with CUDA events on
 * the handle's stream and accumulates device milliseconds per family (read
 * after the solve).  Families: 0 A v products (a5), 1 A^T u products (a1),
 * 2 CGS sweep p1, 3 p2, 4 p3, 5 normalize, 6 small SVD (a7), 7 residuals,
 * 8 recombination (a8/a9), 9 restart misc, 10 collectives, 11 fused CGS2,
 * 12 partial re-orthogonalization decisions (reorth = 1).
 * enable: 0 off, 1 every family, < 0 only the families of the bitmask -enable
 * (fewer event records inside a timed region).  enable resets the counters.
 * ms / calls: host arrays of 16 entries. */
#define SVDSC_PROF_FAMILIES 16
SVDSC_API svdsc_status svdsc_profile_enable(svdsc_handle *h, int enable);
SVDSC_API svdsc_status svdsc_profile_read(const svdsc_handle *h, double *ms, int64_t *calls);

/* ---- kernel-schedule policy --------------------------------------------------
 * The library picks each kernel from the operand's shape (value 0 = automatic,
 * the default and the product path).  A policy forces one schedule so that every
 * kernel the automatic choice can pick is testable at any size; a forced kernel
 * that cannot run a given shape falls back to the always-applicable path
 * (split sweeps / one-CTA Jacobi).  Per handle; applies to the handle's later
 * calls, including matrix analysis (SVDSC_POLICY_SPMV is read there).
 *   SVDSC_POLICY_SPMV:      0 auto (row-length bins for small operands and
 *                           near-uniform rows of >= 48 nonzeros, else register-
 *                           segmented chunks), 1 row-length bins, 2 segmented chunks
 *   SVDSC_POLICY_CGS2:      0 auto (cluster for bases <= 2 MB, else Q-resident
 *                           when the rows fit in shared memory, else streaming),
 *                           1 split sweeps, 2 Q-resident, 3 cp.async streaming,
 *                           4 TMA streaming, 5 thread-block cluster, 6 peer
 *                           (the multi-GPU kernel with in-kernel all-reduces,
 *                           also at P = 1 with a communicator), 7 phased (P > 1:
 *                           three launches with NCCL all-reduces between them);
 *                           set it identically on every rank
 *   SVDSC_POLICY_SMALL_SVD: 0 auto (register Jacobi for p <= 64, else cluster
 *                           block Jacobi + rotation replay), 1 one-CTA Jacobi,
 *                           2 register Jacobi (p <= 64, else auto), 3 cluster
 *                           block Jacobi + rotation replay
 *   SVDSC_POLICY_DEFER:     0 auto (the streaming CGS2 defers its second update
 *                           into the next same-side sweep, DESIGN.md reading
 *                           G5), 1 off (three sweeps per half-step, as written
 *                           in PAPER.md:121; for A/B measurements)
 * EINVAL for an unknown key or value. */
#define SVDSC_POLICY_SPMV 0
#define SVDSC_POLICY_CGS2 1
#define SVDSC_POLICY_SMALL_SVD 2
#define SVDSC_POLICY_DEFER 3
SVDSC_API svdsc_status svdsc_set_policy(svdsc_handle *h, int32_t key, int32_t value);

/* ---- multi-GPU (row-partitioned A) -------------------------- */
/* Rank 0 creates an NCCL unique id (128 bytes, host) that the caller
 * broadcasts (e.g. torch.distributed.broadcast); every rank then calls
 * svdsc_comm_init collectively.  NCCL is loaded at run time (libnccl.so.2);
 * SVDSC_ENCCL if unavailable. */
SVDSC_API svdsc_status svdsc_comm_unique_id(unsigned char id[128]);
SVDSC_API svdsc_status svdsc_comm_init(svdsc_handle *h, int nranks, int rank, const unsigned char id[128]);
/* Collective self-check of the handle's communicator (NCCL or loopback group;
 * call on every rank): one all-gather, reduce-scatter, all-reduce (fp64,
 * rank-dependent integers, exact) and the status all-reduce(min), results
 * compared on the host.  SVDSC_EINVAL without a communicator, SVDSC_ENCCL on a
 * failed call or a wrong sum.  Not needed before a solve; a cheap way to fail
 * fast on a broken NVLink / NCCL setup (bench.py calls it after init). */
SVDSC_API svdsc_status svdsc_comm_check(svdsc_handle *h);
/* In-process ("loopback") group: nranks (<= 16) ranks that are threads of this
 * process, each with its own handle and stream (on one device, or on devices
 * with peer access enabled by the caller).  Each rank's thread calls
 * svdsc_comm_init_group(h, g, rank), then every rank calls the same
 * svdsc_solve concurrently.  Collectives synchronize the rank's stream, meet
 * the other ranks at a host barrier and sum in rank order (bitwise identical
 * on every rank); no kernel waits on another rank.  A testing and
 * single-process backend of the same multi-rank path as NCCL.  The group is
 * reference counted: svdsc_group_destroy may be called once every rank has
 * called svdsc_comm_init_group. */
typedef struct svdsc_group svdsc_group;
SVDSC_API svdsc_status svdsc_group_create(int nranks, svdsc_group **g);
SVDSC_API void svdsc_group_destroy(svdsc_group *g);
SVDSC_API svdsc_status svdsc_comm_init_group(svdsc_handle *h, svdsc_group *g, int rank);
/* Host-only partitioner (no GPU needed): contiguous row blocks of a CSR
 * matrix (host row_ptr, m+1 entries) balanced by the per-step byte cost
 * w_r = 24 nnz_r + 24 basis_cols.  bounds: host,
 * nparts+1 entries, bounds[0] = 0, bounds[nparts] = m. */
SVDSC_API svdsc_status svdsc_partition_rows(int64_t m, const int64_t *row_ptr, int64_t basis_cols,
                                  int nparts, int64_t *bounds);

#ifdef __cplusplus
}
#endif
#endif /* SVDSC_H */
