// internal.h -- private declarations of libsvdsc (B200 / sm_100a).
//
// Layout in HBM:
//   U basis  m_local x (t+1) column-major, ld = roundup(m_local, 32)
//   V basis  n_local x (t+1) column-major, ld = roundup(n_local, 32)
//   T        (t+1) x (t+1) column-major (device, Alg. 2 step 9 layout)
//   every reduction is two-level and deterministic: per-CTA partials stored
//   [column][block], reduced in fixed order by the last CTA to finish.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/svdsc.h"

namespace svdsc {

constexpr int kMaxBlocks = 1184;  // 8 x 148: max CTAs contributing partials
constexpr int kWarp = 32;

// Device-resident control block (one per solve workspace).
struct Ctrl {
    double amax[2];       // largest accepted alpha/beta so far (ring by check parity)
    double inv;           // 1 / norm of the vector being normalized
    int abort;            // != 0: breakdown pending; step kernels are no-ops
    int abort_check;      // check index that broke down
    int abort_kind;       // 0 breakdown (reading Q7); 1 explicit norm needed (multi-GPU CGS2, reading G1)
    int svd_status;       // 0 ok, SVDSC_ESVD_NOCONV
    int svd_sweeps;
    int converged;
    int rankdef;
    double max_resid;
    double svd_tiny;      // p eps ||T||_F: numerically zero column norm (reading Q10b)
    unsigned int cnt[16]; // last-block counters (one per reduction site)
    unsigned int gflags[kMaxBlocks];  // grid-barrier flags of the fused kernels
    // partial re-orthogonalization (reorth = 1, pro.cu)
    int pro_gate;                     // 1: the current half-step re-orthogonalizes
    int pro_force[2];                 // V / U side: next vector re-orthogonalized regardless
    long long pro_reorths;            // half-steps re-orthogonalized so far
};

// ---- CSR operand (device) prepared by analysis --------------------------------
struct CsrOp {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    const int64_t *row_ptr = nullptr;  // nrows+1
    const int32_t *col = nullptr;      // nnz
    const double *val = nullptr;       // nnz
    // row bins: rows grouped by length class, one list per kernel variant
    int32_t *bin_rows = nullptr;       // concatenated row lists
    int64_t bin_off[8] = {0};          // offsets into bin_rows; bin b = [off[b], off[b+1])
    bool bin_identity[8] = {false};    // bin b holds all rows (in order): rows[g] == g
    // long rows (> kLongRow nnz) split into chunks
    int32_t *long_rows = nullptr;      // row id per long row
    int64_t *chunk_first = nullptr;    // first chunk index per long row (+1 sentinel)
    int32_t *chunk_row = nullptr;      // long-row slot per chunk
    int64_t n_long = 0, n_chunks = 0;
    double *chunk_partial = nullptr;   // n_chunks
    // register-segmented schedule ("seg", matvec.cu k_spmv_seg): chunks of
    // kSegChunk consecutive nonzeros, a contiguous run of chunks per warp
    uint32_t *seg_bits = nullptr;      // ceil(nnz/32) words: bit j of word w set <=> nonzero 32w+j starts its row
    int32_t *seg_rows = nullptr;       // the non-empty rows, ascending (row of the k-th row start)
    int32_t *seg_cstart = nullptr;     // per chunk: row starts among the nonzeros before it
    int32_t *seg_empty = nullptr;      // the empty rows (y = -c yprev)
    int64_t seg_nempty = 0, seg_nchunks = 0;
    int seg_cpw = 0, seg_nranges = 0, seg_grid = 0;  // chunks per warp, warp ranges, CTAs
    double *seg_head = nullptr, *seg_tail = nullptr;  // per warp range partial row sums
    unsigned int *seg_flag = nullptr;  // per warp range: 1 once its partial is published (reset by the joiner)
    bool seg = false;                  // use the seg schedule for this operand
    std::vector<void *> owned;         // allocations owned by this operand
    cudaStream_t free_stream = nullptr;  // stream of its pool allocations (g_pool at analysis)
    bool pooled = false;
};
#ifndef SVDSC_SEG_K
#define SVDSC_SEG_K 4
#endif
constexpr int kSegK = SVDSC_SEG_K;     // consecutive nonzeros per lane of a seg chunk (4 or 8)
constexpr int kSegChunk = 32 * kSegK;  // nonzeros per seg chunk

struct DenseOp {
    int64_t nrows = 0, ncols = 0, ld = 0;
    const double *data = nullptr;
    double *partial = nullptr;         // split-K partial sums
    int splits_n = 1, splits_t = 1;
};

void csr_analyze(CsrOp &op, cudaStream_t s);       // bins + long-row chunks
void csr_transpose(const CsrOp &a, CsrOp &at, cudaStream_t s);  // device CSC -> CSR of A^T
void csr_free(CsrOp &op);
// multi-GPU: split a rank's rows by column into loc (columns [c0, c1), rebased)
// and rem (the rest, global columns); both analysed (bins / seg tables)
void csr_split_columns(const CsrOp &a, int64_t c0, int64_t c1, CsrOp &loc, CsrOp &rem, cudaStream_t s);
// rows [r0, r1) of `a` as a standalone operand (rebased row pointers, shared
// column / value arrays); multi-GPU Aᵀu per owner slice
void csr_row_slice(const CsrOp &a, int64_t r0, int64_t r1, CsrOp &out, cudaStream_t s);

// y = A x - c yprev (c = *c_dev if c_dev, else 0).  abort: skip if *abort.
void spmv_csr(const CsrOp &A, const double *x, double *y, const double *c_dev,
              const double *yprev, const int *abort, cudaStream_t s);
void gemv_n(const DenseOp &A, const double *x, double *y, const double *c_dev,
            const double *yprev, const int *abort, cudaStream_t s);
void gemv_t(const DenseOp &A, const double *x, double *y, const double *c_dev,
            const double *yprev, const int *abort, cudaStream_t s);

// ---- CGS2 sweeps (column-major basis Q, N rows, ncols active columns) ----------
struct RedBuf {
    double *partial;      // (kMaxCols) x kMaxBlocks, [col][block]
    int pstride;          // = kMaxBlocks
    double *h1, *h2, *nrm;// reduced outputs (device)
    unsigned int *cnt;    // counters (Ctrl::cnt)
};
int cgs_blocks(int64_t N, int num_sms);
// h1 = Q^T w
void cgs_p1(int64_t N, int ncols, const double *Q, int64_t ldq, const double *w,
            const RedBuf &r, const int *abort, int nsm, cudaStream_t s);
// w <- w - Q h1 (in place), h2 = Q^T w, nrm[0] = ||w||^2
void cgs_p2(int64_t N, int ncols, const double *Q, int64_t ldq, double *w,
            const RedBuf &r, const int *abort, int nsm, cudaStream_t s);
// w <- w - Q h (h = r.h2, or `h` if given), nrm[0] = ||w||^2 (ncols may be 0)
void cgs_p3(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *h,
            const RedBuf &r, const int *abort, int nsm, cudaStream_t s);
// Finalize the norm of a freshly orthogonalized vector (check index `check`):
//   nrm = sqrt(r.nrm[0]); breakdown if nrm <= 1e-14 max(amax, 1) (reading Q7);
//   T entry *t_entry = nrm (or 0 and ctrl->abort = 1 on breakdown);
//   w /= nrm unless breakdown.  force: no breakdown test, T entry untouched.
void normalize(int64_t N, double *w, const RedBuf &r, Ctrl *ctrl, double *t_entry, int check,
               int force, int nsm, cudaStream_t s);
// breakdown replacement vector (counter RNG, bit-exact with the oracle's definition)
void breakdown_vector(int64_t N, int64_t row_offset, double *w, uint64_t seed, uint64_t stream,
                      cudaStream_t s);
// deterministic N(0,1) start vector (library default when v0 == NULL)
void random_start(int64_t N, int64_t row_offset, double *w, uint64_t seed, cudaStream_t s);
void axpy_dev(int64_t N, double *y, const double *c_dev, const double *x, const int *abort,
              cudaStream_t s);  // y -= c x

// Fused single-kernel CGS2 + norm + normalize (single GPU, cooperative launch).
// A dense product left as split-K partials: w[r] = sum_q partial[q*N + r] - c*yprev[r]
// (the k_split_reduce epilogue), to be finished by the CGS2 kernel that reads w.
struct PreReduce {
    const double *partial = nullptr;
    int splits = 0;
    const double *c_dev = nullptr;
    const double *yprev = nullptr;
};
void split_reduce(int64_t N, const PreReduce &pr, double *y, const int *abort, cudaStream_t s);
void gemv_n_partial(const DenseOp &A, const double *x, PreReduce &pr, const double *c_dev, const double *yprev,
                    const int *abort, cudaStream_t s);
void gemv_t_partial(const DenseOp &A, const double *x, PreReduce &pr, const double *c_dev, const double *yprev,
                    const int *abort, cudaStream_t s);

// Deferred second update of the streaming CGS2 (single GPU, DESIGN.md 7
// "deferred sweep C"): a call that defers leaves w' (after the first pass) in
// its basis column and records the second-pass coefficients h2 and 1/beta here;
// the SpMV that follows reads xs = w' / beta, and the next call on the same
// side (or flush_deferred) forms the column's final value
// (w' - Q[:, 0:col] h2) / beta while streaming the same tiles.
constexpr int kDeferMaxCols = 1032;
struct DeferState {
    int flag;     // 1: column `col` of this side still holds w' (pending)
    int col;
    double rbeta;
    double h[kDeferMaxCols];
};
// materialize a pending column (no-op if none): one sweep over its basis
void flush_deferred(int64_t N, double *Q, int64_t ldq, DeferState *st, int nsm, cudaStream_t s);

struct FusedScratch {
    double *partial;      // >= 2*nsm x (ncols+2)
    double *h1, *h2, *h3; // >= ncols+2
    unsigned int *flags;  // >= 2*nsm grid-barrier flags, zeroed once per solve
    unsigned int epoch;   // unique increasing base per launch (multiple of 16)
    const PreReduce *pre = nullptr;  // pending dense split-K reduction of w (or NULL)
    // partial re-orthogonalization (reorth = 1): the launch does its work only
    // if *gate == gate_want (device flag written by pro_decide); else every CTA
    // returns right after preparing the next barrier slot
    const int *gate = nullptr;
    int gate_want = 1;
    // deferred second update (streaming kernel only): st = this side's state
    // (its pending column, if flagged, is formed in the first sweep; with defer,
    // this call leaves its own column pending and writes xs = w' / beta);
    // *deferred (host) reports whether the launch took the deferring path
    DeferState *defer_st = nullptr;
    double *xs = nullptr;
    bool *deferred = nullptr;
    bool maybe_pending = false;  // host: the previous call on this side deferred
};
// false: the fused path is not applicable (caller uses cgs_p1/p2/p3 + normalize)
// tmap: optional CUtensorMap (128 B) of Q for the TMA streaming variant
// (make_basis_tmap), or NULL
bool cgs2_fused(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
                const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nsm, cudaStream_t s,
                const void *tmap);
// Peer mailbox of one rank for the in-kernel one-shot all-reduces of the
// multi-GPU CGS2 (cgs2_peer).  Lives in device memory.  Rank r
// owns `mbox` = [2 parities][P slots][PS doubles] and two arrival counters; the
// CGS2 kernel of rank q writes its column sums of reduction rs into slot
// [rs & 1][q] of EVERY rank's mailbox (NVLink P2P stores through mbox_peer),
// then adds 1 per CTA to every rank's counter [rs & 1] (red.release.sys); a CTA
// proceeds once its own counter [rs & 1] holds ((rs + 1) / 2) * expect arrivals
// and sums the P slots in rank order (bitwise identical on every rank, and
// equal to the loopback backend's rank-ordered sums).  `seq` = reductions
// completed so far on this rank; the counters and seq are zeroed at solve start
// before the status agreement, which all ranks pass only after every rank has
// zeroed (no arrival of the new solve can be lost).
constexpr int kMaxPeers = 8;
struct PeerArgs {
    int P, rank;
    int PS;                // slot stride in doubles (>= ncols + 1 of any call)
    unsigned int expect;   // arrivals per reduction: P x CTAs per rank
    double *mbox;          // this rank's mailbox [2][P][PS]
    unsigned int *ctr;     // this rank's counters [2] (followed by seq)
    unsigned int *seq;     // reductions completed on this rank
    double *mbox_peer[kMaxPeers];       // rank q's mailbox, mapped in this rank's address space
    unsigned int *ctr_peer[kMaxPeers];  // rank q's counters
};
// device bytes of one rank's mailbox block (counters, seq, slots) for P ranks
size_t peer_mailbox_bytes(int P, int PS);
// offsets inside that block
constexpr size_t kPeerHdrBytes = 256;  // ctr[2], seq, padding; slots follow

struct Comm;
// P > 1, peer-memory backend: the whole CGS2 in ONE launch of the streaming
// kernel, its two reductions (and the explicit norm, reading G3) completed
// across the ranks inside the kernel through the peer mailboxes (no NCCL call,
// no host round trip).  peer: device PeerArgs of this rank; nb: CTAs per rank
// (identical on every rank).  false: not applicable.
bool cgs2_peer(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
               const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nb, cudaStream_t s,
               const PeerArgs *peer);
// test support (svdsc_op_cgs2_peer_emulate): P ranks emulated as P groups of
// CTAs of ONE cooperative launch on one GPU, each group with its own operands,
// scratch, control block and peer mailbox (mailboxes of the other groups as
// its peers): the protocol of cgs2_peer without kernels that wait on other
// launches.  grp: device array of P argument blocks prepared by
// cgs2_peer_emulate_prepare.
struct PeerEmuRank {
    int64_t N;
    const double *Q;
    int64_t ldq;
    double *w;
    FusedScratch fs;
    Ctrl *ctrl;
    double *t_entry;
    const PeerArgs *peer;
};
bool cgs2_peer_emulate(int P, int ncols, const PeerEmuRank *ranks, int nb, void *grp_dev, cudaStream_t s);
size_t cgs2_peer_emulate_grp_bytes(int P);
// P > 1: the streaming CGS2 in three launches with the cross-rank all-reduces of
// h1 and [h2; ||w'||^2] between them; *launches is the per-solve fused-launch
// counter (grid-barrier slot chain).  false: not applicable.
bool cgs2_phased(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
                 const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nsm, cudaStream_t s,
                 Comm *comm, unsigned int *launches);
// TMA descriptor of a column-major basis (N rows, ncols_total columns, ld):
// 16 x 16 boxes, SWIZZLE_128B, zero fill beyond N.  Returns false if the
// driver entry point is unavailable.
bool make_basis_tmap(void *map128, const double *base, int64_t N, int64_t ncols_total, int64_t ld);


// partial re-orthogonalization (pro.cu; Q20).  mu/nu: device rows of
// length t+2; part: >= nsm doubles of scratch.  pro_decide writes
// ctrl->pro_gate for the half-step (side 0: v_i from x, side 1: u_i from x);
// kr is the arrow column of T (k after a restart, -1 in the first pass).
void pro_init(int t, double *mu, double *nu, cudaStream_t s);
void pro_decide(int side, int64_t N, const double *x, int i, int kr, const double *T, int ldt, double *mu,
                double *nu, double *part, Ctrl *ctrl, int nsm, cudaStream_t s);
void pro_restart(int t, int k, const double *Vh, int ldvh, double *mu, double *nu, Ctrl *ctrl, cudaStream_t s);

// ---- small SVD / restart ---------------------------------------------------------
// Jacobi SVD of the p x p matrix stored (ld p) in W; outputs Uh, Sh, Vh (ld p),
// writes ctrl->svd_status / svd_sweeps.  Vw is scratch (p x p).  kneed: number
// of leading columns whose zero-sigma completion is required.
// tlog: rotation log of small_svd_log_doubles(p) doubles (NULL: one-CTA
// global-memory Jacobi without the cluster/log path)
size_t small_svd_log_doubles(int p);
void small_svd(int p, const double *Tsrc, int ldt, double *W, double *Vw, double *Uh, double *Sh,
               double *Vh, int kneed, Ctrl *ctrl, const int *abort, double *tlog, cudaStream_t s);
// Eq. (4) residuals, convergence flag (Alg. 2 step 5)
void residuals(int t, int k, const double *T, int ldt, const double *Uh, const double *Sh,
               double tol, double *resid, Ctrl *ctrl, const int *abort, cudaStream_t s);
// Alg. 2 step 9: rho = beta_t Uh(t,1:k); T = 0; T(j,j) = Sh_j; T(j,k) = rho_j
void restart_T(int t, int k, double *T, int ldt, const double *Uh, const double *Sh,
               double *rho, cudaStream_t s);
void recombine(int64_t N, int t, int k, const double *Q, int64_t ldq, const double *W, int ldw,
               double *Qout, int64_t ldo, int nsm, cudaStream_t s);
void copy_col(int64_t N, const double *src, double *dst, cudaStream_t s);
void fill_zero(double *p, int64_t n, cudaStream_t s);

// ---- collectives of the row-partitioned solve (comm.cu) ---------
struct CommError : std::runtime_error {
    svdsc_status st;
    CommError(svdsc_status s, const std::string &m) : std::runtime_error(m), st(s) {}
};
struct Comm {
    int nranks = 1, rank = 0;
    virtual ~Comm() {}
    // enqueued on s (NCCL) or completed before return (loopback)
    virtual void allreduce_sum(double *buf, size_t n, cudaStream_t s) = 0;
    virtual void reduce_scatter_sum(const double *in, double *out, size_t n_each, cudaStream_t s) = 0;
    // sum of every rank's in[0, n) into out on rank `root` only (out ignored elsewhere)
    virtual void reduce_sum(const double *in, double *out, size_t n, int root, cudaStream_t s) = 0;
    virtual void allgather(const double *in, double *out, size_t n_each, cudaStream_t s) = 0;
    // blocking: the minimum of v over the ranks (status agreement before compute)
    virtual int allreduce_min_int(int v, cudaStream_t s) = 0;
    virtual void abort() {}  // a rank failed mid-solve: release the others (loopback)
    // peer mailboxes of the in-kernel all-reduces (cgs2_peer).  peer_setup is
    // collective (every rank, same point, after the status agreement): the first
    // call allocates and exchanges the mailboxes, later calls return the same
    // device PeerArgs; NULL on every rank when any rank cannot map its peers (or
    // the backend has none: loopback, whose ranks share one GPU and must not run
    // kernels that wait on one another).  peer_reset zeroes this rank's counters
    // and seq on s; called at solve start BEFORE the status agreement.
    virtual const PeerArgs *peer_setup(int nsm, cudaStream_t s) { return nullptr; }
    virtual void peer_reset(cudaStream_t s) {}
};
// one-shot peer exchange self-check (svdsc_comm_check): every rank pushes
// (rank + 1) (j + 1) for j < n through the mailboxes; out[j] = the rank-ordered
// sum (device, n <= PS).  Advances seq like one CGS2 reduction.
void peer_check(const PeerArgs *peer, int n, double *out, Ctrl *ctrl, cudaStream_t s);
constexpr int kPeerPS = 1032;  // slot stride: >= t + 2 for t <= 1023
bool comm_nccl_available();
void comm_nccl_unique_id(unsigned char id[128]);
Comm *comm_nccl_create(const unsigned char id[128], int nranks, int rank);
struct LoopbackGroup;
LoopbackGroup *loopback_group_create(int nranks);
void loopback_group_release(LoopbackGroup *g);
Comm *comm_loopback_create(LoopbackGroup *g, int rank);

// ---- kernel-schedule policy (svdsc_set_policy, include/svdsc.h) -----------------
// 0 everywhere = automatic choice by shape (the product default).  Set per call
// from the handle (thread-local: distinct handles on distinct threads are
// independent); tests use it to run every schedule the automatic choice may pick.
struct Policy {
    int spmv = 0;       // SVDSC_POLICY_SPMV
    int cgs2 = 0;       // SVDSC_POLICY_CGS2
    int small_svd = 0;  // SVDSC_POLICY_SMALL_SVD
    int defer = 0;      // SVDSC_POLICY_DEFER
};
extern thread_local Policy g_policy;

// ---- matrix analysis allocations -------------------------------------------------
// Set by the C ABI around matrix analysis: the handle's private memory pool and
// stream, so derived structures (CSC copy, bins, seg tables) and the analysis
// temporaries come from pooled memory (a host-buffer solve creates and
// destroys its matrix every call: cudaMalloc / cudaFree of the 1.8 GB CSC copy
// of BASELINE config 4 cost tens of ms each time).  NULL: cudaMalloc.
extern thread_local cudaMemPool_t g_pool;
extern thread_local cudaStream_t g_pool_stream;
void *analysis_alloc(size_t bytes);
void analysis_free(void *p);

// ---- launch bookkeeping ----------------------------------------------------------
extern thread_local int64_t g_launches;
inline void count_launch() { ++g_launches; }

// Programmatic dependent launch (PDL): a kernel launched by launch_pdl may be
// scheduled while its stream predecessor is still draining (onto the SMs that
// predecessor leaves idle); it runs only work that reads nothing the
// predecessor writes (e.g. staging the basis Q), then pdl_wait() -- which
// returns once the predecessor grid has completed and its writes are visible
// -- before anything else.  pdl_trigger(), issued after the wait, lets the
// successor launch early in turn.  A kernel that never calls pdl_wait must not
// be launched with launch_pdl.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    int na = 1;
    if (cluster > 1) {
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = cluster;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        na = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

}  // namespace svdsc

#define SVDSC_CUDA_CHECK_LAUNCH() ::svdsc::count_launch()
