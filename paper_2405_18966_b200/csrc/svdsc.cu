// svdsc.cu -- C ABI (include/svdsc.h) and the host driver of Alg. 2.
//
// The host issues every kernel of a pass asynchronously on the handle's stream
// and synchronizes ONCE per pass (to read the convergence flag of Alg. 2
// step 5).  Data-dependent rare events (Lanczos breakdown,
// DESIGN.md reading Q7) do not need a per-step sync: the normalizing kernel
// raises a device flag, every later kernel of the pass becomes a no-op, and
// the host repairs the broken vector at the pass-end sync and resumes.
//
// Multi-GPU: A is row-partitioned; U rows follow A's rows;
// V is split into equal slices of n_pad / P rows.  Per Lanczos step:
// reduce-scatter of the partial A^T u, all-gather of v_{i+1}, and two
// all-reduces per re-orthogonalization (h1, then [h2; ||w'||^2]) between the
// three launches of the streaming CGS2 kernel (comm.cu: NCCL, or the
// in-process loopback backend).  Every rank agrees on the call's status
// (all-reduce of min) before any compute.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"

using namespace svdsc;

namespace {
struct SvdscError : std::runtime_error {
    svdsc_status st;
    SvdscError(svdsc_status s, const std::string &m) : std::runtime_error(m), st(s) {}
};

inline void ck(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw SvdscError(SVDSC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
inline void einval(bool bad, const std::string &m) {
    if (bad) throw SvdscError(SVDSC_EINVAL, m);
}
}  // namespace

// per-family CUDA-event timing (svdsc_profile_enable)
struct Prof {
    bool on = false;
    unsigned mask = 0xffffffffu;  // families recorded
    double ms[SVDSC_PROF_FAMILIES] = {0};
    int64_t calls[SVDSC_PROF_FAMILIES] = {0};
    struct Pair {
        cudaEvent_t a, b;
        int fam;
    };
    std::vector<Pair> pending, pool;
    int open_fam = -1;
    cudaEvent_t open_ev = nullptr;
    cudaEvent_t take() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back().a;
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void begin(int fam, cudaStream_t s) {
        if (!on || !((mask >> fam) & 1u)) return;
        open_fam = fam;
        open_ev = take();
        cudaEventRecord(open_ev, s);
    }
    void end(cudaStream_t s) {
        if (!on || open_fam < 0) return;
        cudaEvent_t e = take();
        cudaEventRecord(e, s);
        pending.push_back({open_ev, e, open_fam});
        open_fam = -1;
    }
    void harvest() {  // after a stream sync
        for (auto &p : pending) {
            float t = 0.f;
            if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
                ms[p.fam] += t;
                calls[p.fam]++;
            } else {
                cudaGetLastError();
            }
            pool.push_back({p.a, nullptr, 0});
            pool.push_back({p.b, nullptr, 0});
        }
        pending.clear();
    }
    ~Prof() {
        for (auto &p : pending) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        for (auto &p : pool) cudaEventDestroy(p.a);
    }
};

struct svdsc_handle {
    Prof prof;
    int device = 0, nsm = 148;
    cudaStream_t stream = nullptr;
    std::string err;
    Comm *comm = nullptr;        // multi-rank collectives (comm.cu); NULL: single rank
    int nranks = 1, rank = 0;
    Policy policy;               // kernel-schedule policy (svdsc_set_policy)
    cudaMemPool_t pool = nullptr;  // private pool of the library's stream-ordered allocations
    cudaStream_t cap = nullptr;    // graph-capture stream (the caller's may be the uncapturable legacy stream)
    Ctrl *hctrl = nullptr;       // pinned host mirror of the control block
    void *scratch = nullptr;     // op-level scratch
    size_t scratch_bytes = 0;
    // P > 1: stream of the v all-gather that overlaps the local-column product
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_v = nullptr, ev_g = nullptr;
};

struct svdsc_group {
    LoopbackGroup *g;
    int P;
    int nranks() const { return P; }
};

struct svdsc_matrix {
    svdsc_handle *h = nullptr;
    int kind = 0;  // 0 CSR, 1 dense
    int64_t m_local = 0, n = 0, row_offset = 0, m_global = 0, nnz = 0;
    CsrOp A, At;
    // P > 1 (CSR): A split by column into the rank's own slice of v (Aloc,
    // rebased columns) and the rest (Arem), so A v overlaps the all-gather
    bool split = false;
    int split_P = 0;
    CsrOp Aloc, Arem;
    // P > 1 (CSR): the CSC copy cut into the owners' slices of Aᵀu, so each
    // slice's reduction to its owner overlaps the next slice's product
    std::vector<CsrOp> AtS;
    DenseOp D;
    double *dense_partial = nullptr;
    double seconds_analysis = 0.0;  // host wall time of svdsc_matrix_* (validation, bins, CSC)
};

namespace {

template <typename F>
svdsc_status guarded(svdsc_handle *h, F &&f) {
    if (h) g_policy = h->policy;
    try {
        f();
        return SVDSC_OK;
    } catch (const SvdscError &e) {
        if (h) h->err = e.what();
        return e.st;
    } catch (const CommError &e) {
        if (h) h->err = e.what();
        return e.st;
    } catch (const std::exception &e) {
        if (h) h->err = e.what();
        return SVDSC_ECUDA;
    }
}

int64_t roundup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// validation kernels (contract checks before any compute)
__global__ void k_validate_csr(int64_t m, int64_t n, int64_t nnz, const int64_t *rp, const int32_t *col,
                               const double *val, int *bad) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = tid; r < m; r += stride)
        if (rp[r + 1] < rp[r]) atomicOr(bad, 1);
    for (int64_t p = tid; p < nnz; p += stride) {
        if (col[p] < 0 || col[p] >= n) atomicOr(bad, 2);
        if (!isfinite(val[p])) atomicOr(bad, 4);
    }
    if (tid == 0 && (rp[0] != 0 || rp[m] != nnz)) atomicOr(bad, 8);
}

__global__ void k_validate_dense(int64_t m, int64_t n, int64_t ld, const double *a, int *bad) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < m * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx % m, c = idx / m;
        if (!isfinite(a[r + c * ld])) atomicOr(bad, 4);
    }
}

// V(:, 0:k) of every rank's slice, gathered slice-major -> column-major n x k
void copy_gathered(const double *tmp, int64_t ns, int k, int P, int64_t n, double *V, int64_t ldv, cudaStream_t s) {
    for (int q = 0; q < P; q++) {
        const int64_t rows = std::min(ns, n - q * ns);
        if (rows <= 0) continue;
        ck(cudaMemcpy2DAsync(V + q * ns, ldv * sizeof(double), tmp + (int64_t)q * ns * k, ns * sizeof(double),
                             rows * sizeof(double), k, cudaMemcpyDeviceToDevice, s),
           "memcpy2D");
    }
}

// ---------------------------------------------------------------------------
// workspace
struct Ws {
    double *U = nullptr, *V = nullptr, *T = nullptr;
    double *W = nullptr, *Vw = nullptr, *Uh = nullptr, *Vh = nullptr, *Sh = nullptr;
    double *partial = nullptr, *h1 = nullptr, *h2 = nullptr, *nrm = nullptr, *rho = nullptr, *resid = nullptr;
    double *yfull = nullptr, *vfull = nullptr, *vtmp = nullptr;
    double *tlog = nullptr;
    double *pro_mu = nullptr, *pro_nu = nullptr, *pro_part = nullptr;  // reorth = 1 (pro.cu)
    Ctrl *ctrl = nullptr;
    int64_t ldu = 0, ldv = 0, nv = 0, n_pad = 0;
    double *cm1 = nullptr;  // P > 1: the constant -1 (z += Arem v_full as z = Arem v_full - (-1) z)
    // deferred second update of the streaming CGS2 (P = 1): per
    // side (0 = V, 1 = U) the pending-column state and the next product's input
    DeferState *dst[2] = {nullptr, nullptr};
    double *xs[2] = {nullptr, nullptr};
    int ldt = 0;
};

struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(size_t n) {
        off = roundup((int64_t)off, 256);
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += std::max<size_t>(n, 1) * sizeof(T);
        return p;
    }
};

size_t carve(Ws &w, void *base, int64_t m, int64_t n, int t, int k, int P) {
    Carver c{reinterpret_cast<char *>(base)};
    w.n_pad = roundup(n, P);
    w.nv = w.n_pad / P;
    w.ldu = roundup(std::max<int64_t>(m, 1), 32);
    w.ldv = roundup(std::max<int64_t>(w.nv, 1), 32);
    w.ldt = t + 1;
    w.ctrl = c.take<Ctrl>(1);
    w.U = c.take<double>((size_t)w.ldu * (t + 1));
    w.V = c.take<double>((size_t)w.ldv * (t + 1));
    w.T = c.take<double>((size_t)(t + 1) * (t + 1));
    w.W = c.take<double>((size_t)t * t);
    w.Vw = c.take<double>((size_t)t * t);
    w.Uh = c.take<double>((size_t)t * t);
    w.Vh = c.take<double>((size_t)t * t);
    w.Sh = c.take<double>(t);
    w.partial = c.take<double>((size_t)(t + 2) * kMaxBlocks);
    w.h1 = c.take<double>(t + 2);
    w.h2 = c.take<double>(t + 2);
    w.nrm = c.take<double>(4);
    w.rho = c.take<double>(k);
    w.resid = c.take<double>(k);
    w.tlog = c.take<double>(small_svd_log_doubles(t));
    w.pro_mu = c.take<double>(t + 2);
    w.pro_nu = c.take<double>(t + 2);
    w.pro_part = c.take<double>(kMaxBlocks);
    w.dst[0] = c.take<DeferState>(1);
    w.dst[1] = c.take<DeferState>(1);
    w.xs[0] = c.take<double>(roundup(std::max<int64_t>(w.nv, 1), 32));
    w.xs[1] = c.take<double>(roundup(std::max<int64_t>(m, 1), 32));
    if (P > 1) {
        w.yfull = c.take<double>(w.n_pad);
        w.vfull = c.take<double>(w.n_pad);
        w.vtmp = c.take<double>((size_t)w.n_pad * k);
        w.cm1 = c.take<double>(1);
    }
    return c.off + 256;
}

int resolve_t(const svdsc_opts *o, int64_t m_global, int64_t n) {
    int64_t t = o->t > 0 ? o->t : std::max<int64_t>(15, 3 * (int64_t)o->k);
    t = std::min<int64_t>(t, std::min(m_global, n) - 1);
    return (int)t;
}

void check_opts(const svdsc_matrix *M, const svdsc_opts *o) {
    einval(!o, "opts is NULL");
    einval(o->k < 1, "k must be >= 1");
    einval(!(o->tol > 0.0), "tol must be > 0");
    const int t = resolve_t(o, M->m_global, M->n);
    einval(t < o->k + 2, "subspace dimension t = min(max(15,3k), min(m,n)-1) < k+2 (SPEC.md:309)");
    einval(t > 1023, "t > 1023 is not supported");
    einval(o->reorth < -1 || o->reorth > 2, "reorth must be -1, 0, 1 or 2");
}

// stream-ordered allocation from the handle's private pool
void *pool_alloc(svdsc_handle *H, size_t bytes, cudaStream_t s) {
    void *p = nullptr;
    ck(cudaMallocFromPoolAsync(&p, std::max<size_t>(bytes, 8), H->pool, s), "cudaMallocFromPoolAsync");
    return p;
}

// ---------------------------------------------------------------------------
// the solver for one call
struct Solver {
    svdsc_matrix *M;
    svdsc_handle *H;
    const svdsc_opts *o;
    Ws w;
    RedBuf rb;
    cudaStream_t s;
    int t, k, P, rank, nsm;
    int64_t m, nv, n;
    const int *abort;
    int64_t matvecs = 0, steps = 0, breakdowns = 0, bytes_model = 0, bytes_reorth = 0;
    uint64_t bd_stream = 0;
    int check = 0;
    int64_t bytesA = 0;

    // ---- collectives (no-ops for P = 1) ----
    void allreduce(double *buf, size_t count) {
        if (P > 1) H->comm->allreduce_sum(buf, count, s);
    }

    // z = A x - c zprev on the local rows (x = V column slice)
    void Av(const double *vcol, double *z, const double *c_dev, const double *zprev) {
        const double *x = vcol;
        if (P > 1 && M->split && M->split_P == P) {
            // the all-gather of v runs on the comm stream while
            // the rank's own columns are multiplied (z = Aloc v_slice - c zprev),
            // then z += Arem v_full (c = -1, in place)
            ck(cudaEventRecord(H->ev_v, s), "event");
            ck(cudaStreamWaitEvent(H->comm_stream, H->ev_v, 0), "wait");
            H->comm->allgather(vcol, w.vfull, (size_t)nv, H->comm_stream);
            ck(cudaEventRecord(H->ev_g, H->comm_stream), "event");
            H->prof.begin(0, s);
            spmv_csr(M->Aloc, vcol, z, c_dev, zprev, abort, s);
            ck(cudaStreamWaitEvent(s, H->ev_g, 0), "wait");
            spmv_csr(M->Arem, w.vfull, z, w.cm1, z, abort, s);
            H->prof.end(s);
            matvecs++;
            return;
        }
        if (P > 1) {
            H->comm->allgather(vcol, w.vfull, (size_t)nv, s);
            x = w.vfull;
        }
        H->prof.begin(0, s);
        if (M->kind == 0) spmv_csr(M->A, x, z, c_dev, zprev, abort, s);
        else if (defer_reduce()) gemv_n_partial(M->D, x, pending, c_dev, zprev, abort, s);
        else gemv_n(M->D, x, z, c_dev, zprev, abort, s);
        H->prof.end(s);
        matvecs++;
    }
    // dense single-GPU products leave their split-K partials for the fused CGS2
    // kernel, which finishes the reduction while staging w (one launch less per
    // half-step); any other consumer calls finish_pending() first
    PreReduce pending;
    bool defer_reduce() const { return M->kind == 1 && P == 1 && fused_ok && o->reorth == 2; }
    void finish_pending(int64_t N, double *wv) {
        if (pending.partial) {
            split_reduce(N, pending, wv, abort, s);
            pending = PreReduce{};
        }
    }
    // wslice = (A^T u)_slice - c wprev
    void Atu(const double *u, double *wcol, const double *c_dev, const double *wprev) {
        if (P == 1) {
            H->prof.begin(1, s);
            if (M->kind == 0) spmv_csr(M->At, u, wcol, c_dev, wprev, abort, s);
            else if (defer_reduce()) gemv_t_partial(M->D, u, pending, c_dev, wprev, abort, s);
            else gemv_t(M->D, u, wcol, c_dev, wprev, abort, s);
            H->prof.end(s);
        } else if (M->kind == 0 && (int)M->AtS.size() == P && H->comm_stream) {
            // the owners' slices of Aᵀu in owner order; slice
            // q's reduction to rank q (comm stream) overlaps slice q+1's product
            H->prof.begin(1, s);
            for (int q = 0; q < P; q++) {
                double *yq = w.yfull + (int64_t)q * nv;
                if (M->AtS[(size_t)q].nrows > 0) spmv_csr(M->AtS[(size_t)q], u, yq, nullptr, nullptr, abort, s);
                ck(cudaEventRecord(H->ev_v, s), "event");
                ck(cudaStreamWaitEvent(H->comm_stream, H->ev_v, 0), "wait");
                H->comm->reduce_sum(yq, wcol, (size_t)nv, q, H->comm_stream);
            }
            ck(cudaEventRecord(H->ev_g, H->comm_stream), "event");
            ck(cudaStreamWaitEvent(s, H->ev_g, 0), "wait");
            H->prof.end(s);
            if (c_dev) axpy_dev(nv, wcol, c_dev, wprev, abort, s);
        } else {
            if (M->kind == 0) spmv_csr(M->At, u, w.yfull, nullptr, nullptr, abort, s);
            else gemv_t(M->D, u, w.yfull, nullptr, nullptr, abort, s);
            H->comm->reduce_scatter_sum(w.yfull, wcol, (size_t)nv, s);
            if (c_dev) axpy_dev(nv, wcol, c_dev, wprev, abort, s);
        }
        matvecs++;
    }
    // two-pass CGS against Q(:, 0:ncols) then ||w||^2 in rb.nrm
    void cgs2(int64_t N, int ncols, const double *Q, int64_t ldq, double *wv, bool force_reorth) {
        if (ncols > 0 && (o->reorth != 0 || force_reorth)) {
            H->prof.begin(2, s);
            cgs_p1(N, ncols, Q, ldq, wv, rb, abort, nsm, s);
            H->prof.end(s);
            allreduce(rb.h1, ncols);
            H->prof.begin(3, s);
            cgs_p2(N, ncols, Q, ldq, wv, rb, abort, nsm, s);
            H->prof.end(s);
            allreduce(rb.h2, ncols + 1);
            H->prof.begin(4, s);
            cgs_p3(N, ncols, Q, ldq, wv, rb.h2, rb, abort, nsm, s);
            H->prof.end(s);
        } else {
            H->prof.begin(4, s);
            cgs_p3(N, 0, Q, ldq, wv, nullptr, rb, abort, nsm, s);
            H->prof.end(s);
        }
        allreduce(rb.nrm, 1);
    }

    bool fused_ok = true;
    unsigned int fused_launches = 0;
    // peer mailboxes of the in-kernel all-reduces (NCCL backend, P > 1, or
    // SVDSC_POLICY_CGS2 = 6 with a one-rank communicator); NULL: not used
    const PeerArgs *peer = nullptr;
    // deferred second update (P = 1, full CGS2): maypend[side] = the last column
    // written on that side was left pending (its product input is w.xs[side]);
    // pend_cols[side] = that column's index (for the byte model of the flush)
    bool maypend[2] = {false, false};
    int pend_cols[2] = {0, 0};
    // single GPU, or the multi-GPU peer kernel (the phased / loopback path keeps
    // the three sweeps)
    bool defer_ok() const { return o->reorth == 2 && (P == 1 || peer) && g_policy.defer == 0; }
    // form pending columns (pass end: the small SVD's recombination and the
    // restart read the bases; flush kernels are no-ops if the device shows none)
    void flush_pending() {
        const int64_t Ns[2] = {nv, m};
        double *base[2] = {w.V, w.U};
        const int64_t ld[2] = {w.ldv, w.ldu};
        for (int sd = 0; sd < 2; sd++) {
            if (!maypend[sd]) continue;
            flush_deferred(Ns[sd], base[sd], ld[sd], w.dst[sd], nsm, s);
            bytes_model += 8 * Ns[sd] * ((int64_t)pend_cols[sd] + 2);
            maypend[sd] = false;
        }
    }
    alignas(64) unsigned char tmapU[128], tmapV[128];
    bool have_tmap = false;
    // re-orthogonalize wv against Q(:, 0:ncols) (optionally after wv -= Q pre_h),
    // then beta = ||wv||, breakdown test, T entry, wv /= beta.
    // side: 0 = V, 1 = U (deferred second update), -1 = none.  Returns whether
    // the call left its column pending (the product reads w.xs[side])
    bool last_deferred = false;
    void orth_norm(int64_t N, int ncols, const double *Q, int64_t ldq, double *wv, double *t_entry, int chk,
                   const double *pre_h, int side = -1) {
        last_deferred = false;
        if (peer && o->reorth != 0 && fused_ok) {
            // one launch: CGS2 + norm + normalization with the cross-rank
            // reductions completed inside the kernel
            FusedScratch fs{w.partial, w.h1, w.h2, w.nrm, w.ctrl->gflags, 16u * (++fused_launches), nullptr};
            bool dflag = false;
            if (side >= 0 && defer_ok()) {
                fs.defer_st = w.dst[side];
                fs.xs = w.xs[side];
                fs.deferred = &dflag;
                fs.maybe_pending = maypend[side];
            }
            if (pending.partial) finish_pending(N, wv);
            H->prof.begin(11, s);
            const bool ok = cgs2_peer(N, ncols, Q, ldq, wv, pre_h, fs, w.ctrl, t_entry, chk, nsm, s, peer);
            H->prof.end(s);
            if (side >= 0) {
                if (maypend[side]) bytes_model += 8 * N, bytes_reorth += 8 * N;
                maypend[side] = ok && dflag;
                if (dflag) pend_cols[side] = ncols;
            }
            if (ok) {
                last_deferred = dflag;
                return;
            }
            // not applicable (identical shapes on every rank: every rank falls back)
            --fused_launches;
        }
        if (P == 1 && o->reorth != 0 && fused_ok) {
            FusedScratch fs{w.partial, w.h1, w.h2, w.nrm, w.ctrl->gflags, 16u * (++fused_launches),
                            pending.partial ? &pending : nullptr};
            bool dflag = false;
            if (side >= 0 && defer_ok()) {
                fs.defer_st = w.dst[side];
                fs.xs = w.xs[side];
                fs.deferred = &dflag;
                fs.maybe_pending = maypend[side];
            }
            H->prof.begin(11, s);
            const void *tm = have_tmap ? (Q == w.U ? (const void *)tmapU : (Q == w.V ? (const void *)tmapV : nullptr))
                                       : nullptr;
            const bool ok = cgs2_fused(N, ncols, Q, ldq, wv, pre_h, fs, w.ctrl, t_entry, chk, nsm, s, tm);
            H->prof.end(s);
            if (side >= 0) {  // a pending input column was formed (or flushed) by this call
                if (maypend[side]) bytes_model += 8 * N, bytes_reorth += 8 * N;
                maypend[side] = ok && dflag;
                if (dflag) pend_cols[side] = ncols;
            }
            if (ok) {
                pending = PreReduce{};
                last_deferred = dflag;
                return;
            }
            fused_ok = false;
        }
        if (P > 1 && o->reorth != 0 && fused_ok) {
            FusedScratch fs{w.partial, w.h1, w.h2, w.nrm, w.ctrl->gflags, 0u, nullptr};
            H->prof.begin(11, s);
            const bool ok = cgs2_phased(N, ncols, Q, ldq, wv, pre_h, fs, w.ctrl, t_entry, chk, nsm, s, H->comm,
                                        &fused_launches);
            H->prof.end(s);
            if (ok) return;
            fused_ok = false;
        }
        finish_pending(N, wv);
        if (pre_h) cgs_p3(N, ncols, Q, ldq, wv, pre_h, rb, abort, nsm, s);
        cgs2(N, ncols, Q, ldq, wv, false);
        H->prof.begin(5, s);
        normalize(N, wv, rb, w.ctrl, t_entry, chk, 0, nsm, s);
        H->prof.end(s);
    }

    // partial re-orthogonalization (reorth = 1, Q20): the decision
    // kernel sets ctrl->pro_gate; the full CGS2 launch runs iff it is 1, the
    // normalize-only launch (ncols = 0) iff it is 0
    int pro_kr = -1;        // arrow column of T: k after the first restart
    int64_t reorth_halves = 0;
    void orth_norm_pro(int side, int i, int64_t N, const double *Q, int64_t ldq, double *wv, double *t_entry,
                       int chk) {
        einval(!fused_ok, "reorth = 1 needs the fused CGS2 kernels (SVDSC_NO_FUSED is set)");
        finish_pending(N, wv);
        H->prof.begin(12, s);
        pro_decide(side, N, wv, i, pro_kr, w.T, w.ldt, w.pro_mu, w.pro_nu, w.pro_part, w.ctrl, nsm, s);
        H->prof.end(s);
        H->prof.begin(11, s);
        const void *tm = have_tmap ? (Q == w.U ? (const void *)tmapU : (Q == w.V ? (const void *)tmapV : nullptr))
                                   : nullptr;
        for (int want = 1; want >= 0; want--) {
            FusedScratch fs{w.partial, w.h1, w.h2, w.nrm, w.ctrl->gflags, 16u * (++fused_launches), nullptr,
                            &w.ctrl->pro_gate, want};
            if (!cgs2_fused(N, want ? i : 0, Q, ldq, wv, nullptr, fs, w.ctrl, t_entry, chk, nsm, s, tm))
                throw SvdscError(SVDSC_EINVAL, "reorth = 1: fused CGS2 path not applicable");
        }
        H->prof.end(s);
    }

    double *Ucol(int j) { return w.U + (int64_t)j * w.ldu; }
    double *Vcol(int j) { return w.V + (int64_t)j * w.ldv; }
    double *Tm(int i, int j) { return w.T + i + (int64_t)j * w.ldt; }

    // half-steps: 0 start (u_1), 1 V side of step i, 2 U side of step i, 3 restart u_{k+1}
    struct Half {
        int kind, i;
    };

    void run_half(const Half &h, int chk) {
        switch (h.kind) {
            case 0:  // Alg. 1 lines 2-3
                Av(Vcol(0), Ucol(0), nullptr, nullptr);
                orth_norm(m, 0, w.U, w.ldu, Ucol(0), Tm(0, 0), chk, nullptr, 1);
                bytes_model += bytesA + 8 * m * 5;
                bytes_reorth += 8 * m * 5;
                break;
            case 1: {  // Alg. 1 lines 5-6 + re-orthogonalization
                const int i = h.i;
                // a pending u_i / v_i: the product reads w' / beta
                Atu(maypend[1] ? w.xs[1] : Ucol(i - 1), Vcol(i), Tm(i - 1, i - 1),
                    maypend[0] ? w.xs[0] : Vcol(i - 1));
                if (o->reorth == 1) {
                    orth_norm_pro(0, i, nv, w.V, w.ldv, Vcol(i), Tm(i - 1, i), chk);
                } else {
                    orth_norm(nv, i, w.V, w.ldv, Vcol(i), Tm(i - 1, i), chk, nullptr, 0);
                    reorth_halves += o->reorth == 2;
                }
                steps++;
                const int64_t cb = 8 * nv * ((last_deferred ? 2 : 3) * (int64_t)i + 5);
                bytes_model += bytesA + cb;
                if (o->reorth == 2) bytes_reorth += cb;
                break;
            }
            case 2: {  // Alg. 1 lines 7-8 + re-orthogonalization
                const int i = h.i;
                Av(maypend[0] ? w.xs[0] : Vcol(i), Ucol(i), Tm(i - 1, i), maypend[1] ? w.xs[1] : Ucol(i - 1));
                if (o->reorth == 1) {
                    orth_norm_pro(1, i, m, w.U, w.ldu, Ucol(i), Tm(i, i), chk);
                } else {
                    orth_norm(m, i, w.U, w.ldu, Ucol(i), Tm(i, i), chk, nullptr, 1);
                    reorth_halves += o->reorth == 2;
                }
                const int64_t cb = 8 * m * ((last_deferred ? 2 : 3) * (int64_t)i + 5);
                bytes_model += bytesA + cb;
                if (o->reorth == 2) bytes_reorth += cb;
                break;
            }
            case 3: {  // Alg. 2 steps 10-11: u_{k+1} = A v_{k+1} - Uk rho, re-orth
                Av(Vcol(k), Ucol(k), nullptr, nullptr);
                orth_norm(m, k, w.U, w.ldu, Ucol(k), Tm(k, k), chk, w.rho, 1);
                // the product, the Ũ_k rho sweep and the CGS2 against Ũ_k
                const int64_t cb = 8 * m * ((last_deferred ? 3 : 4) * (int64_t)k + 5);
                bytes_model += bytesA + cb;
                if (o->reorth != 0) bytes_reorth += cb;
                break;
            }
        }
    }

    // breakdown repair (reading Q7): replacement vector, CGS2, normalize
    void fix(const Half &h) {
        double *col;
        const double *Q;
        int64_t N, ldq, off;
        int ncols;
        if (h.kind == 1) {
            col = Vcol(h.i), Q = w.V, N = nv, ldq = w.ldv, ncols = h.i, off = (int64_t)rank * nv;
        } else {
            const int j = h.kind == 0 ? 0 : (h.kind == 2 ? h.i : k);
            col = Ucol(j), Q = w.U, N = m, ldq = w.ldu, ncols = j, off = M->row_offset;
        }
        const int64_t valid = (h.kind == 1) ? std::max<int64_t>(0, std::min(nv, n - off)) : N;
        if (valid < N) ck(cudaMemsetAsync(col + valid, 0, (N - valid) * sizeof(double), s), "memset");
        breakdown_vector(valid, off, col, o->seed, bd_stream++, s);
        cgs2(N, ncols, Q, ldq, col, true);
        normalize(N, col, rb, w.ctrl, nullptr, 0, 1, nsm, s);
        breakdowns++;
    }

    // multi-GPU CGS2 whose second pass removed more than half of ||w'||^2 (reading
    // G1): w'' is formed; its explicit norm (one more all-reduce), the breakdown
    // test, the T entry and the normalization, as the single-GPU kernel does
    void fix_norm(const Half &h, int chk) {
        double *col, *tent;
        int64_t N;
        if (h.kind == 1) {
            col = Vcol(h.i), N = nv, tent = Tm(h.i - 1, h.i);
        } else {
            const int j = h.kind == 0 ? 0 : (h.kind == 2 ? h.i : k);
            col = Ucol(j), N = m, tent = Tm(j, j);
        }
        cgs2(N, 0, nullptr, 0, col, false);
        normalize(N, col, rb, w.ctrl, tent, chk, 0, nsm, s);
    }

    Ctrl read_ctrl() {
        ck(cudaMemcpyAsync(H->hctrl, w.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s), "D2H ctrl");
        ck(cudaStreamSynchronize(s), "sync");
        ck(cudaGetLastError(), "kernels");
        H->prof.harvest();
        return *H->hctrl;
    }

    // runs the plan from pos; handles breakdowns; returns with the pass complete
    // enqueue the plan's half-steps [pos, end) and, for a full pass, the small
    // SVD and the convergence test.  Check indices are relative to the plan
    // (plans have an even number of half-steps, so the amax ring parity of
    // reading Q7 is unchanged), which makes a restart pass's kernel sequence
    // identical from pass to pass: it is captured once into a CUDA graph and
    // replayed (one launch per pass instead of one per kernel).
    void enqueue_plan(const std::vector<Half> &plan, size_t pos, bool with_svd) {
        for (size_t idx = pos; idx < plan.size(); idx++) run_half(plan[idx], (int)idx);
        // pending columns are formed before anything reads the bases (a
        // breakdown's repair, the restart's recombination, the final assembly)
        flush_pending();
        if (with_svd) {
            H->prof.begin(6, s);
            small_svd(t, w.T, w.ldt, w.W, w.Vw, w.Uh, w.Sh, w.Vh, k, w.ctrl, abort, w.tlog, s);
            H->prof.end(s);
            H->prof.begin(7, s);
            residuals(t, k, w.T, w.ldt, w.Uh, w.Sh, o->tol, w.resid, w.ctrl, abort, s);
            H->prof.end(s);
        }
    }

    cudaGraphExec_t gexec = nullptr;  // the restart pass (captured at its first use)
    bool graph_ok = true;
    unsigned int graph_launch_base = 0;  // fused-launch counter at the capture's start
    int64_t graph_kernels = 0, graph_bytes_model = 0, graph_bytes_reorth = 0, graph_matvecs = 0, graph_steps = 0,
            graph_reorth_halves = 0;

    bool replay_restart_plan(const std::vector<Half> &plan) {
        // (not while profiling: event records inside a stream capture failed on
        // this driver -- cudaErrorIllegalState -- so profiled solves run eagerly)
        if (!graph_ok || P != 1 || H->prof.on) return false;
        if (!gexec) {
            // capture: the barrier-slot ring is zeroed at the graph's start, so a
            // replay does not depend on the slots the previous launches left
            const unsigned int fl0 = fused_launches;
            const int64_t l0 = g_launches, b0 = bytes_model, r0 = bytes_reorth, mv0 = matvecs, st0 = steps,
                          rh0 = reorth_halves;
            if (!H->cap && cudaStreamCreateWithFlags(&H->cap, cudaStreamNonBlocking) != cudaSuccess) {
                cudaGetLastError();
                graph_ok = false;
                return false;
            }
            const cudaStream_t s_user = s;
            s = H->cap;  // enqueue into the capture
            if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                cudaGetLastError();
                s = s_user;
                graph_ok = false;
                return false;
            }
            bool ok = true;
            try {
                fused_launches = 0;
                ck(cudaMemsetAsync(w.ctrl->gflags, 0, sizeof(w.ctrl->gflags), s), "memset slots");
                enqueue_plan(plan, 0, true);
            } catch (...) {
                ok = false;
            }
            cudaGraph_t g = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(s, &g);
            s = s_user;
            if (ok && ec == cudaSuccess && g && cudaGraphInstantiate(&gexec, g, 0) == cudaSuccess) {
                cudaGraphDestroy(g);
            } else {
                if (g) cudaGraphDestroy(g);
                gexec = nullptr;
                cudaGetLastError();
                graph_ok = false;
                fused_launches = fl0;
                g_launches = l0, bytes_model = b0, bytes_reorth = r0, matvecs = mv0, steps = st0;
                reorth_halves = rh0;
                return false;
            }
            graph_launch_base = fused_launches;  // launches inside the graph (from 0)
            fused_launches = fl0;  // nothing ran yet: the host bookkeeping is redone per replay below
            graph_kernels = g_launches - l0;
            graph_bytes_model = bytes_model - b0, graph_bytes_reorth = bytes_reorth - r0;
            graph_matvecs = matvecs - mv0, graph_steps = steps - st0, graph_reorth_halves = reorth_halves - rh0;
            g_launches = l0, bytes_model = b0, bytes_reorth = r0, matvecs = mv0, steps = st0, reorth_halves = rh0;
        }
        ck(cudaGraphLaunch(gexec, s), "cudaGraphLaunch");
        // the graph's launches used barrier slots 1..graph_launch_base and zeroed
        // the next one: eager launches after it continue from there
        fused_launches = graph_launch_base;
        g_launches += graph_kernels;
        bytes_model += graph_bytes_model, bytes_reorth += graph_bytes_reorth;
        matvecs += graph_matvecs, steps += graph_steps, reorth_halves += graph_reorth_halves;
        return true;
    }

    // runs the plan; handles breakdowns; returns with the pass complete
    void run_plan(const std::vector<Half> &plan, bool with_svd, bool restart_plan) {
        size_t pos = 0;
        for (;;) {
            if (!(pos == 0 && restart_plan && with_svd && replay_restart_plan(plan)))
                enqueue_plan(plan, pos, with_svd);
            Ctrl c = read_ctrl();
            if (!c.abort) return;
            const int idx = c.abort_check;
            if (c.abort_kind == 2)
                throw CommError(SVDSC_ENCCL, "multi-GPU CGS2: a peer rank did not arrive at an in-kernel all-reduce");
            if (c.abort_kind == 3) throw SvdscError(SVDSC_ECUDA, "deferred CGS2 update: pending column mismatch");
            if (idx < 0 || idx >= (int)plan.size()) throw SvdscError(SVDSC_ECUDA, "breakdown bookkeeping");
            const int zero[2] = {0, 0};
            ck(cudaMemcpyAsync(&w.ctrl->abort, &zero[0], sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
            ck(cudaMemcpyAsync(&w.ctrl->abort_kind, &zero[1], sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
            if (c.abort_kind == 1) fix_norm(plan[idx], idx);
            else fix(plan[idx]);
            pos = idx + 1;
        }
    }

    ~Solver() {
        if (gexec) cudaGraphExecDestroy(gexec);
    }

    svdsc_status solve(void *ws_base, double *S, double *Uout, int64_t ldu_out, double *Vout, int64_t ldv_out,
                       double *resid, svdsc_info *info, bool lbp_only, double *Tout) {
        const int maxit = o->maxit > 0 ? o->maxit : 10;
        carve(w, ws_base, m, n, t, k, P);
        nv = w.nv;
        rb = RedBuf{w.partial, kMaxBlocks, w.h1, w.h2, w.nrm, w.ctrl->cnt};
        fused_ok = true;
        // TMA descriptors of the bases (used by the TMA streaming CGS2 kernel,
        // SVDSC_POLICY_CGS2 = 4)
        have_tmap = g_policy.cgs2 == 4 && make_basis_tmap(tmapU, w.U, m, t + 1, w.ldu) &&
                    make_basis_tmap(tmapV, w.V, nv, t + 1, w.ldv);
        abort = &w.ctrl->abort;
        bytesA = M->kind == 0 ? 12 * M->nnz + 4 * (m + 1) : 8 * m * n;
        ck(cudaMemsetAsync(w.ctrl, 0, sizeof(Ctrl), s), "memset");
        ck(cudaMemsetAsync(w.T, 0, sizeof(double) * (t + 1) * (t + 1), s), "memset");
        ck(cudaMemsetAsync(w.dst[0], 0, sizeof(DeferState), s), "memset");
        ck(cudaMemsetAsync(w.dst[1], 0, sizeof(DeferState), s), "memset");
        maypend[0] = maypend[1] = false;
        if (o->reorth == 1) pro_init(t, w.pro_mu, w.pro_nu, s);
        if (P > 1) {
            static const double minus_one = -1.0;
            ck(cudaMemcpyAsync(w.cm1, &minus_one, sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
            if ((M->split || !M->AtS.empty()) && !H->comm_stream) {
                ck(cudaStreamCreateWithFlags(&H->comm_stream, cudaStreamNonBlocking), "stream");
                ck(cudaEventCreateWithFlags(&H->ev_v, cudaEventDisableTiming), "event");
                ck(cudaEventCreateWithFlags(&H->ev_g, cudaEventDisableTiming), "event");
            }
            ck(cudaMemsetAsync(w.V, 0, sizeof(double) * w.ldv * (t + 1), s), "memset");
            ck(cudaMemsetAsync(w.yfull, 0, sizeof(double) * w.n_pad, s), "memset");
        }
        if (lbp_only) ck(cudaMemsetAsync(w.U, 0, sizeof(double) * w.ldu * (t + 1), s), "memset");
        // Alg. 1 line 1: v_1 = v0 / ||v0||
        const int64_t off = (int64_t)rank * nv, valid = std::max<int64_t>(0, std::min(nv, n - off));
        if (o->v0) {
            if (valid > 0)
                ck(cudaMemcpyAsync(Vcol(0), o->v0 + off, valid * sizeof(double), cudaMemcpyDeviceToDevice, s), "v0");
        } else {
            random_start(valid, off, Vcol(0), o->seed, s);
        }
        cgs2(nv, 0, w.V, w.ldv, Vcol(0), false);
        double nv0 = 0.0;
        ck(cudaMemcpyAsync(&nv0, w.nrm, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
        einval(!(nv0 > 0.0) || !std::isfinite(nv0), "start vector v0 is zero or not finite");
        normalize(nv, Vcol(0), rb, w.ctrl, nullptr, 0, 1, nsm, s);

        std::vector<Half> plan;
        plan.push_back({0, 0});
        for (int i = 1; i <= t; i++) {
            plan.push_back({1, i});
            if (i < t) plan.push_back({2, i});  // u_{t+1} is not needed (reading Q2)
        }
        int passes = 0;
        Ctrl c{};
        if (lbp_only) {
            run_plan(plan, false, false);
            for (int j = 0; j <= t; j++) {
                ck(cudaMemcpyAsync(Uout + (int64_t)j * ldu_out, Ucol(j), m * sizeof(double), cudaMemcpyDeviceToDevice, s),
                   "copy U");
                ck(cudaMemcpyAsync(Vout + (int64_t)j * ldv_out, Vcol(j), n * sizeof(double), cudaMemcpyDeviceToDevice, s),
                   "copy V");
            }
            ck(cudaMemcpyAsync(Tout, w.T, sizeof(double) * (t + 1) * (t + 1), cudaMemcpyDeviceToDevice, s), "copy T");
            ck(cudaStreamSynchronize(s), "sync");
            passes = 1;
        } else {
            for (;;) {
                run_plan(plan, true, passes > 0);
                c = *H->hctrl;
                if (c.svd_status != 0) throw SvdscError(SVDSC_ESVD_NOCONV, "small Jacobi SVD did not converge in 50 sweeps");
                if (c.rankdef) throw SvdscError(SVDSC_ERANKDEF, "zero Ritz value with non-negligible residual");
                passes++;
                const bool stop = o->fixed_passes > 0 ? passes >= o->fixed_passes : (c.converged || passes >= maxit);
                if (stop) break;
                // augmented restart, Alg. 2 steps 8-12
                H->prof.begin(8, s);
                recombine(m, t, k, w.U, w.ldu, w.Uh, t, w.U, w.ldu, nsm, s);
                recombine(nv, t, k, w.V, w.ldv, w.Vh, t, w.V, w.ldv, nsm, s);
                H->prof.end(s);
                H->prof.begin(9, s);
                copy_col(nv, Vcol(t), Vcol(k), s);  // v_{k+1} = v_{t+1}
                restart_T(t, k, w.T, w.ldt, w.Uh, w.Sh, w.rho, s);
                if (o->reorth == 1) {
                    pro_restart(t, k, w.Vh, t, w.pro_mu, w.pro_nu, w.ctrl, s);
                    pro_kr = k;
                }
                H->prof.end(s);
                matvecs += 0;
                plan.clear();
                plan.push_back({3, 0});
                for (int i = k + 1; i <= t; i++) {
                    plan.push_back({1, i});
                    if (i < t) plan.push_back({2, i});
                }
            }
            // Alg. 2 steps 15-16: S, U_k = U(:,1:t) Uh(:,1:k), V_k likewise
            ck(cudaMemcpyAsync(S, w.Sh, k * sizeof(double), cudaMemcpyDeviceToDevice, s), "S");
            if (resid) ck(cudaMemcpyAsync(resid, w.resid, k * sizeof(double), cudaMemcpyDeviceToDevice, s), "resid");
            H->prof.begin(8, s);
            recombine(m, t, k, w.U, w.ldu, w.Uh, t, Uout, ldu_out, nsm, s);
            H->prof.end(s);
            if (P == 1) {
                recombine(nv, t, k, w.V, w.ldv, w.Vh, t, Vout, ldv_out, nsm, s);
            } else {
                recombine(nv, t, k, w.V, w.ldv, w.Vh, t, w.vtmp + (int64_t)rank * nv * k, nv, nsm, s);
                H->comm->allgather(w.vtmp + (int64_t)rank * nv * k, w.vtmp, (size_t)nv * k, s);
                copy_gathered(w.vtmp, nv, k, P, n, Vout, ldv_out, s);
            }
            ck(cudaStreamSynchronize(s), "sync");
            ck(cudaGetLastError(), "final");
        }
        if (info) {
            info->passes = passes;
            info->restarts = std::max(0, passes - 1);
            info->converged = lbp_only ? 0 : c.converged;
            info->t_used = t;
            info->steps = steps;
            info->matvecs = matvecs;
            info->breakdowns = breakdowns;
            info->max_resid = lbp_only ? 0.0 : c.max_resid;
            info->bytes_model = bytes_model;
            info->bytes_reorth = bytes_reorth;
            info->reorths = o->reorth == 1 ? H->hctrl->pro_reorths : reorth_halves;
        }
        if (!lbp_only && !c.converged) return SVDSC_NOT_CONVERGED;
        return SVDSC_OK;
    }
};

svdsc_status run_solver(svdsc_matrix *M, const svdsc_opts *o_in, void *ws, size_t ws_bytes, double *S, double *U,
                        int64_t ldu, double *V, int64_t ldv, double *resid, svdsc_info *info, bool lbp_only,
                        int t_override, double *Tout) {
    svdsc_handle *H = M->h;
    svdsc_status ret = SVDSC_OK;
    const int64_t l0 = g_launches;
    auto t0 = std::chrono::steady_clock::now();
    svdsc_opts oo{};
    Solver sv{};
    size_t need = 0;
    // contract checks (no device work), then every rank agrees on the status
    svdsc_status st = guarded(H, [&] {
        einval(!o_in, "opts is NULL");
        oo = *o_in;
        if (!lbp_only) check_opts(M, &oo);
        einval(oo.reorth < -1 || oo.reorth > 2, "reorth must be -1, 0, 1 or 2");
        // 0 (a zero-initialized struct) = the paper's method, CGS2 every half-step;
        // -1 = re-orthogonalization off (test only); internally 2 / 1 / 0
        oo.reorth = oo.reorth == 0 ? 2 : (oo.reorth < 0 ? 0 : oo.reorth);
        einval(oo.reorth == 1 && H->nranks > 1, "reorth = 1 (partial) is single-GPU only");
        sv.M = M;
        sv.H = H;
        sv.o = &oo;
        sv.s = H->stream;
        sv.k = oo.k;
        sv.t = t_override > 0 ? t_override : resolve_t(&oo, M->m_global, M->n);
        sv.P = H->nranks;
        sv.rank = H->rank;
        sv.nsm = H->nsm;
        sv.m = M->m_local;
        sv.n = M->n;
        einval(!lbp_only && (!S || !U || !V), "S, U and V must be non-NULL");
        einval(!lbp_only && ldu < std::max<int64_t>(1, M->m_local), "ldu < m_local");
        einval(!lbp_only && ldv < std::max<int64_t>(1, M->n), "ldv < ncols");
        Ws probe;
        need = carve(probe, nullptr, M->m_local, M->n, sv.t, sv.k, sv.P);
        einval(ws && ws_bytes < need, "workspace too small (see svdsc_workspace_size)");
    });
    // the peer CGS2 (P > 1 with a backend that maps peer memory, or forced by
    // SVDSC_POLICY_CGS2 = 6): counters zeroed before the status agreement, so
    // no rank's first arrival of this solve can precede another rank's reset
    const bool want_peer = H->comm && oo.reorth == 2 && g_policy.cgs2 != 7 &&
                           (H->nranks > 1 || g_policy.cgs2 == 6);
    if (st == SVDSC_OK && want_peer) st = guarded(H, [&] { H->comm->peer_reset(H->stream); });
    if (H->nranks > 1) {
        int agreed = (int)st;
        const std::string local_err = H->err;
        const svdsc_status sa = guarded(H, [&] { agreed = H->comm->allreduce_min_int((int)st, H->stream); });
        if (sa != SVDSC_OK) return sa;
        if (st != SVDSC_OK) {
            H->err = local_err;
            return st;
        }
        if (agreed != SVDSC_OK) {
            H->err = "another rank rejected the call (status " + std::to_string(agreed) + ")";
            return (svdsc_status)agreed;
        }
    } else if (st != SVDSC_OK) {
        return st;
    }
    st = guarded(H, [&] {
        if (want_peer) sv.peer = H->comm->peer_setup(H->nsm, sv.s);
        void *base = ws;
        const bool own = !base;
        if (own) base = pool_alloc(H, need, sv.s);
        try {
            ret = sv.solve(base, S, U, ldu, V, ldv, resid, info, lbp_only, Tout);
        } catch (...) {
            if (H->comm) H->comm->abort();
            if (own) {
                cudaFreeAsync(base, sv.s);
                cudaStreamSynchronize(sv.s);
            }
            throw;
        }
        if (own) {
            ck(cudaFreeAsync(base, sv.s), "cudaFreeAsync");
            ck(cudaStreamSynchronize(sv.s), "sync");
        }
    });
    if (info) {
        info->seconds_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        info->seconds_analysis = M->seconds_analysis;
        info->launches = g_launches - l0;
    }
    return st != SVDSC_OK ? st : ret;
}

void matrix_common_dense_setup(svdsc_matrix *M) {
    DenseOp &D = M->D;
    const int64_t m = D.nrows, n = D.ncols;
    const int nsm = M->h->nsm;
    const int64_t rb = (m + 63) / 64;
    D.splits_n = (int)std::max<int64_t>(1, std::min<int64_t>(64, ((int64_t)nsm * 8 + rb - 1) / std::max<int64_t>(rb, 1)));
    D.splits_n = (int)std::min<int64_t>(D.splits_n, std::max<int64_t>(1, n / 16));
    const int64_t cb = (n + 7) / 8;  // k_gemv_t: 8 warps x 1 column per CTA
    // ~2500 CTAs (2.8 waves at 6 CTAs/SM): measured best at config 2 (splits 4-5:
    // 120 us vs 127 us at 2 splits; tools/timeline.py sweep)
    D.splits_t = (int)std::max<int64_t>(1, std::min<int64_t>({64, (2500 + cb / 2) / cb, std::max<int64_t>(1, m / 1024)}));
    const size_t need = std::max<size_t>((size_t)D.splits_n * m, (size_t)D.splits_t * n);
    ck(cudaMalloc(&M->dense_partial, need * sizeof(double)), "cudaMalloc");
    D.partial = M->dense_partial;
}

}  // namespace

// ===========================================================================
// C ABI
extern "C" {

const char *svdsc_version(void) { return "svdsc 0.1 sm_100a"; }

svdsc_status svdsc_create(svdsc_handle **h, void *stream) {
    if (!h) return SVDSC_EINVAL;
    *h = nullptr;
    svdsc_handle *H = new svdsc_handle();
    svdsc_status st = guarded(H, [&] {
        ck(cudaGetDevice(&H->device), "cudaGetDevice");
        ck(cudaDeviceGetAttribute(&H->nsm, cudaDevAttrMultiProcessorCount, H->device), "attr");
        H->stream = reinterpret_cast<cudaStream_t>(stream);
        ck(cudaMallocHost(&H->hctrl, sizeof(Ctrl)), "cudaMallocHost");
        // stream-ordered allocations (NULL workspace, host-buffer entry points)
        // come from a private pool that keeps its memory mapped between solves
        // instead of returning it at every synchronization (re-mapping the
        // 800 MB operand of BASELINE config 2 cost ~40 ms per solve); the
        // device's default pool, which the host application may use, is untouched
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = H->device;
        ck(cudaMemPoolCreate(&H->pool, &props), "cudaMemPoolCreate");
        uint64_t keep = UINT64_MAX;
        ck(cudaMemPoolSetAttribute(H->pool, cudaMemPoolAttrReleaseThreshold, &keep), "pool attribute");
    });
    if (st != SVDSC_OK) {
        if (H->hctrl) cudaFreeHost(H->hctrl);
        if (H->pool) cudaMemPoolDestroy(H->pool);
        delete H;
        return st;
    }
    *h = H;
    return SVDSC_OK;
}

svdsc_status svdsc_set_stream(svdsc_handle *h, void *stream) {
    if (!h) return SVDSC_EINVAL;
    h->stream = reinterpret_cast<cudaStream_t>(stream);
    return SVDSC_OK;
}

void svdsc_destroy(svdsc_handle *h) {
    if (!h) return;
    cudaStreamSynchronize(h->stream);
    delete h->comm;
    if (h->cap) cudaStreamDestroy(h->cap);
    if (h->comm_stream) {
        cudaStreamSynchronize(h->comm_stream);
        cudaStreamDestroy(h->comm_stream);
        cudaEventDestroy(h->ev_v);
        cudaEventDestroy(h->ev_g);
    }
    if (h->hctrl) cudaFreeHost(h->hctrl);
    if (h->scratch) cudaFree(h->scratch);
    if (h->pool) cudaMemPoolDestroy(h->pool);
    delete h;
}

const char *svdsc_last_error(const svdsc_handle *h) { return h ? h->err.c_str() : "null handle"; }

svdsc_status svdsc_matrix_csr(svdsc_handle *h, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t *row_ptr,
                              const int32_t *col_idx, const double *values, int64_t row_offset, int64_t m_global,
                              svdsc_matrix **Mout) {
    if (!h || !Mout) return SVDSC_EINVAL;
    *Mout = nullptr;
    svdsc_matrix *M = new svdsc_matrix();
    const auto t0 = std::chrono::steady_clock::now();
    svdsc_status st = guarded(h, [&] {
        einval(nrows < 0 || ncols < 1 || nnz < 0, "bad dimensions");
        einval(!row_ptr || (nnz > 0 && (!col_idx || !values)), "NULL array");
        einval(nnz >= (int64_t)1 << 31 || nrows >= (int64_t)1 << 31 || ncols >= (int64_t)1 << 31,
               "nnz, nrows and ncols must be < 2^31 per rank");
        einval(row_offset < 0 || m_global < row_offset + nrows, "row_offset/m_global inconsistent");
        M->h = h;
        M->kind = 0;
        M->m_local = nrows;
        M->n = ncols;
        M->nnz = nnz;
        M->row_offset = row_offset;
        M->m_global = m_global;
        cudaStream_t s = h->stream;
        int *bad = nullptr;
        bad = (int *)pool_alloc(h, sizeof(int), s);
        ck(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
        k_validate_csr<<<148 * 4, 256, 0, s>>>(nrows, ncols, nnz, row_ptr, col_idx, values, bad);
        int hb = 0;
        ck(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaFreeAsync(bad, s), "free");
        ck(cudaStreamSynchronize(s), "sync");
        einval(hb & 8, "row_ptr[0] != 0 or row_ptr[nrows] != nnz");
        einval(hb & 1, "row_ptr is not monotone");
        einval(hb & 2, "column index out of range");
        einval(hb & 4, "non-finite value");
        M->A.nrows = nrows;
        M->A.ncols = ncols;
        M->A.nnz = nnz;
        M->A.row_ptr = row_ptr;
        M->A.col = col_idx;
        M->A.val = values;
        struct PoolScope {  // analysis allocations from the handle's pool
            PoolScope(cudaMemPool_t p, cudaStream_t st) {
                g_pool = p;
                g_pool_stream = st;
            }
            ~PoolScope() {
                g_pool = nullptr;
                g_pool_stream = nullptr;
            }
        } scope(h->pool, s);
        csr_analyze(M->A, s);
        csr_transpose(M->A, M->At, s);
        if (h->nranks > 1) {
            // the solver's slices of v: nv = ceil(n / P) rows per rank (carve)
            const int64_t P = h->nranks, nv = (ncols + P - 1) / P;
            const int64_t c0 = std::min<int64_t>(ncols, (int64_t)h->rank * nv), c1 = std::min<int64_t>(ncols, c0 + nv);
            if (c1 > c0) {
                csr_split_columns(M->A, c0, c1, M->Aloc, M->Arem, s);
                M->split = true;
                M->split_P = (int)P;
            }
            M->AtS.resize((size_t)P);
            for (int64_t q = 0; q < P; q++) {
                const int64_t r0 = std::min<int64_t>(ncols, q * nv), r1 = std::min<int64_t>(ncols, r0 + nv);
                csr_row_slice(M->At, r0, r1, M->AtS[(size_t)q], s);
            }
        }
        M->seconds_analysis = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
    if (st != SVDSC_OK) {
        csr_free(M->A);
        csr_free(M->At);
        csr_free(M->Aloc);
        csr_free(M->Arem);
        for (CsrOp &op : M->AtS) csr_free(op);
        delete M;
        return st;
    }
    *Mout = M;
    return SVDSC_OK;
}

svdsc_status svdsc_matrix_dense(svdsc_handle *h, int64_t nrows, int64_t ncols, int64_t ld, const double *data,
                                int64_t row_offset, int64_t m_global, svdsc_matrix **Mout) {
    if (!h || !Mout) return SVDSC_EINVAL;
    *Mout = nullptr;
    svdsc_matrix *M = new svdsc_matrix();
    const auto t0 = std::chrono::steady_clock::now();
    svdsc_status st = guarded(h, [&] {
        einval(nrows < 1 || ncols < 1 || ld < nrows, "bad dimensions");
        einval(!data, "NULL data");
        einval(row_offset < 0 || m_global < row_offset + nrows, "row_offset/m_global inconsistent");
        M->h = h;
        M->kind = 1;
        M->m_local = nrows;
        M->n = ncols;
        M->row_offset = row_offset;
        M->m_global = m_global;
        M->nnz = nrows * ncols;
        cudaStream_t s = h->stream;
        int *bad = nullptr;
        bad = (int *)pool_alloc(h, sizeof(int), s);
        ck(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
        k_validate_dense<<<148 * 4, 256, 0, s>>>(nrows, ncols, ld, data, bad);
        int hb = 0;
        ck(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaFreeAsync(bad, s), "free");
        ck(cudaStreamSynchronize(s), "sync");
        einval(hb & 4, "non-finite value");
        M->D.nrows = nrows;
        M->D.ncols = ncols;
        M->D.ld = ld;
        M->D.data = data;
        matrix_common_dense_setup(M);
        M->seconds_analysis = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
    if (st != SVDSC_OK) {
        if (M->dense_partial) cudaFree(M->dense_partial);
        delete M;
        return st;
    }
    *Mout = M;
    return SVDSC_OK;
}

void svdsc_matrix_destroy(svdsc_matrix *M) {
    if (!M) return;
    csr_free(M->A);
    csr_free(M->At);
    csr_free(M->Aloc);
    csr_free(M->Arem);
    for (CsrOp &op : M->AtS) csr_free(op);
    if (M->dense_partial) cudaFree(M->dense_partial);
    delete M;
}

svdsc_status svdsc_workspace_size(svdsc_matrix *M, const svdsc_opts *o, size_t *bytes) {
    if (!M || !bytes) return SVDSC_EINVAL;
    return guarded(M->h, [&] {
        check_opts(M, o);
        Ws w;
        *bytes = carve(w, nullptr, M->m_local, M->n, resolve_t(o, M->m_global, M->n), o->k, M->h->nranks);
    });
}

svdsc_status svdsc_solve(svdsc_matrix *M, const svdsc_opts *o, void *workspace, size_t ws_bytes, double *S, double *U,
                         int64_t ldu, double *V, int64_t ldv, double *resid, svdsc_info *info) {
    if (!M) return SVDSC_EINVAL;
    return run_solver(M, o, workspace, ws_bytes, S, U, ldu, V, ldv, resid, info, false, 0, nullptr);
}

svdsc_status svdsc_op_lbp(svdsc_matrix *M, const svdsc_opts *o, int32_t t, const double *v0, double *U, int64_t ldu,
                          double *V, int64_t ldv, double *T, svdsc_info *info) {
    if (!M || !o) return SVDSC_EINVAL;
    if (M->h->nranks != 1 || t < 1 || t + 1 > std::min(M->m_global, M->n) || t > 1023 || !U || !V || !T ||
        ldu < M->m_local || ldv < M->n) {
        M->h->err = "op_lbp: single rank, 1 <= t <= 1023, t+1 <= min(m,n), non-NULL U, V, T";
        return SVDSC_EINVAL;
    }
    svdsc_opts oo = *o;
    oo.v0 = v0;
    oo.k = 1;
    oo.tol = oo.tol > 0 ? oo.tol : 1e-10;
    return run_solver(M, &oo, nullptr, 0, nullptr, U, ldu, V, ldv, nullptr, info, true, t, T);
}

svdsc_status svdsc_solve_host_csr(svdsc_handle *h, int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr,
                                  const int32_t *col_idx, const double *values, const svdsc_opts *o, double *S,
                                  double *U, double *V, double *resid, svdsc_info *info) {
    if (!h || !o) return SVDSC_EINVAL;
    std::vector<void *> bufs;
    svdsc_matrix *M = nullptr;
    svdsc_status ret = SVDSC_OK;
    svdsc_status st = guarded(h, [&] {
        einval(m < 1 || n < 1 || nnz < 0 || !row_ptr || !S || !U || !V, "bad arguments");
        cudaStream_t s = h->stream;
        auto dalloc = [&](size_t b) {
            void *p = pool_alloc(h, b, s);
            bufs.push_back(p);
            return p;
        };
        int64_t *drp = (int64_t *)dalloc((m + 1) * 8);
        int32_t *dci = (int32_t *)dalloc(nnz * 4);
        double *dva = (double *)dalloc(nnz * 8);
        ck(cudaMemcpyAsync(drp, row_ptr, (m + 1) * 8, cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemcpyAsync(dci, col_idx, nnz * 4, cudaMemcpyHostToDevice, s), "H2D");
        ck(cudaMemcpyAsync(dva, values, nnz * 8, cudaMemcpyHostToDevice, s), "H2D");
        svdsc_opts oo = *o;
        if (o->v0) {
            double *dv0 = (double *)dalloc(n * 8);
            ck(cudaMemcpyAsync(dv0, o->v0, n * 8, cudaMemcpyHostToDevice, s), "H2D");
            oo.v0 = dv0;
        }
        const int k = o->k;
        double *dS = (double *)dalloc(k * 8), *dU = (double *)dalloc(m * k * 8), *dV = (double *)dalloc(n * k * 8),
               *dr = (double *)dalloc(k * 8);
        svdsc_status s1 = svdsc_matrix_csr(h, m, n, nnz, drp, dci, dva, 0, m, &M);
        if (s1 != SVDSC_OK) throw SvdscError(s1, h->err);
        ret = svdsc_solve(M, &oo, nullptr, 0, dS, dU, m, dV, n, dr, info);
        if (ret < 0) throw SvdscError(ret, h->err);
        ck(cudaMemcpyAsync(S, dS, k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(U, dU, m * k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(V, dV, n * k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        if (resid) ck(cudaMemcpyAsync(resid, dr, k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
    });
    svdsc_matrix_destroy(M);
    for (void *p : bufs) cudaFreeAsync(p, h->stream);
    cudaStreamSynchronize(h->stream);
    return st != SVDSC_OK ? st : ret;
}

svdsc_status svdsc_solve_host_dense(svdsc_handle *h, int64_t m, int64_t n, const double *data, const svdsc_opts *o,
                                    double *S, double *U, double *V, double *resid, svdsc_info *info) {
    if (!h || !o) return SVDSC_EINVAL;
    std::vector<void *> bufs;
    svdsc_matrix *M = nullptr;
    svdsc_status ret = SVDSC_OK;
    svdsc_status st = guarded(h, [&] {
        einval(m < 1 || n < 1 || !data || !S || !U || !V, "bad arguments");
        cudaStream_t s = h->stream;
        auto dalloc = [&](size_t b) {
            void *p = pool_alloc(h, b, s);
            bufs.push_back(p);
            return p;
        };
        double *dA = (double *)dalloc((size_t)m * n * 8);
        ck(cudaMemcpyAsync(dA, data, (size_t)m * n * 8, cudaMemcpyHostToDevice, s), "H2D");
        svdsc_opts oo = *o;
        if (o->v0) {
            double *dv0 = (double *)dalloc(n * 8);
            ck(cudaMemcpyAsync(dv0, o->v0, n * 8, cudaMemcpyHostToDevice, s), "H2D");
            oo.v0 = dv0;
        }
        const int k = o->k;
        double *dS = (double *)dalloc(k * 8), *dU = (double *)dalloc(m * k * 8), *dV = (double *)dalloc(n * k * 8),
               *dr = (double *)dalloc(k * 8);
        svdsc_status s1 = svdsc_matrix_dense(h, m, n, m, dA, 0, m, &M);
        if (s1 != SVDSC_OK) throw SvdscError(s1, h->err);
        ret = svdsc_solve(M, &oo, nullptr, 0, dS, dU, m, dV, n, dr, info);
        if (ret < 0) throw SvdscError(ret, h->err);
        ck(cudaMemcpyAsync(S, dS, k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(U, dU, m * k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(V, dV, n * k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        if (resid) ck(cudaMemcpyAsync(resid, dr, k * 8, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
    });
    svdsc_matrix_destroy(M);
    for (void *p : bufs) cudaFreeAsync(p, h->stream);
    cudaStreamSynchronize(h->stream);
    return st != SVDSC_OK ? st : ret;
}

// ---- step-level ops -----------------------------------------------------------
svdsc_status svdsc_op_matvec(svdsc_matrix *M, int trans, const double *x, double *y, const double *c_dev,
                             const double *yprev) {
    if (!M) return SVDSC_EINVAL;
    return guarded(M->h, [&] {
        einval(!x || !y || (c_dev && !yprev), "NULL vector");
        cudaStream_t s = M->h->stream;
        if (M->kind == 0) spmv_csr(trans ? M->At : M->A, x, y, c_dev, yprev, nullptr, s);
        else if (trans) gemv_t(M->D, x, y, c_dev, yprev, nullptr, s);
        else gemv_n(M->D, x, y, c_dev, yprev, nullptr, s);
        ck(cudaGetLastError(), "matvec launch");
    });
}

namespace {
// op-level scratch: ctrl + partials + reductions + Jacobi work arrays
struct OpScratch {
    Ctrl *ctrl;
    double *partial, *h1, *h2, *nrm, *W, *Vw, *tlog;
};
OpScratch op_scratch(svdsc_handle *h, int maxcols, int p) {
    Carver c{nullptr};
    c.take<Ctrl>(1);
    c.take<double>((size_t)(maxcols + 2) * kMaxBlocks);
    c.take<double>(maxcols + 2);
    c.take<double>(maxcols + 2);
    c.take<double>(4);
    c.take<double>((size_t)p * p);
    c.take<double>((size_t)p * p);
    c.take<double>(small_svd_log_doubles(p));
    const size_t need = c.off + 256;
    if (need > h->scratch_bytes) {
        if (h->scratch) cudaFree(h->scratch);
        h->scratch = nullptr;
        ck(cudaMalloc(&h->scratch, need), "cudaMalloc scratch");
        h->scratch_bytes = need;
    }
    Carver d{reinterpret_cast<char *>(h->scratch)};
    OpScratch o;
    o.ctrl = d.take<Ctrl>(1);
    o.partial = d.take<double>((size_t)(maxcols + 2) * kMaxBlocks);
    o.h1 = d.take<double>(maxcols + 2);
    o.h2 = d.take<double>(maxcols + 2);
    o.nrm = d.take<double>(4);
    o.W = d.take<double>((size_t)p * p);
    o.Vw = d.take<double>((size_t)p * p);
    o.tlog = d.take<double>(small_svd_log_doubles(p));
    ck(cudaMemsetAsync(o.ctrl, 0, sizeof(Ctrl), h->stream), "memset");
    return o;
}
}  // namespace

svdsc_status svdsc_op_cgs2(svdsc_handle *h, int64_t N, int64_t ncols, const double *Q, int64_t ldq, double *w,
                           double *norm_dev) {
    if (!h) return SVDSC_EINVAL;
    return guarded(h, [&] {
        einval(N < 1 || ncols < 0 || ncols > 1023 || (ncols > 0 && (!Q || ldq < N)) || !w, "bad arguments");
        OpScratch sc = op_scratch(h, (int)ncols, 1);
        RedBuf rb{sc.partial, kMaxBlocks, sc.h1, sc.h2, sc.nrm, sc.ctrl->cnt};
        cudaStream_t s = h->stream;
        double *tent = sc.nrm + 2;  // the T entry (beta / alpha) of this half-step
        // the solver's kernel for this shape (SVDSC_POLICY_CGS2), else the split sweeps
        alignas(64) unsigned char tm[128];
        const bool have = g_policy.cgs2 == 4 && ncols > 0 && make_basis_tmap(tm, Q, N, ncols, ldq);
        FusedScratch fs{sc.partial, sc.h1, sc.h2, sc.nrm, sc.ctrl->gflags, 16u};
        if (!cgs2_fused(N, (int)ncols, Q, ldq, w, nullptr, fs, sc.ctrl, tent, 0, h->nsm, s, have ? tm : nullptr)) {
            if (ncols > 0) {
                cgs_p1(N, (int)ncols, Q, ldq, w, rb, nullptr, h->nsm, s);
                cgs_p2(N, (int)ncols, Q, ldq, w, rb, nullptr, h->nsm, s);
                cgs_p3(N, (int)ncols, Q, ldq, w, sc.h2, rb, nullptr, h->nsm, s);
            } else {
                cgs_p3(N, 0, Q, ldq, w, nullptr, rb, nullptr, h->nsm, s);
            }
            normalize(N, w, rb, sc.ctrl, tent, 0, 0, h->nsm, s);
        }
        if (norm_dev) ck(cudaMemcpyAsync(norm_dev, tent, sizeof(double), cudaMemcpyDeviceToDevice, s), "D2D");
        ck(cudaStreamSynchronize(s), "sync");
        ck(cudaGetLastError(), "cgs2");
    });
}

svdsc_status svdsc_op_cgs2_peer_emulate(svdsc_handle *h, int32_t P, const int64_t *row0, int64_t ncols,
                                        const double *Q, int64_t ldq, double *w, double *beta_out) {
    if (!h) return SVDSC_EINVAL;
    return guarded(h, [&] {
        einval(P < 1 || P > kMaxPeers || !row0 || !w || !beta_out || ncols < 0 || ncols > 384, "bad arguments");
        einval(row0[0] != 0, "row0[0] must be 0");
        for (int q = 0; q < P; q++)
            einval(row0[q + 1] <= row0[q] || (row0[q] & 1), "row0: ranks need >= 1 row and even offsets");
        const int64_t N = row0[P];
        einval(ncols > 0 && (!Q || ldq < N || (ldq & 1)), "bad basis");
        einval((reinterpret_cast<uintptr_t>(w) & 15) || (ncols > 0 && (reinterpret_cast<uintptr_t>(Q) & 15)),
               "Q and w must be 16-byte aligned");
        const int nb = h->nsm / P;
        einval(nb < 1, "fewer SMs than ranks");
        cudaStream_t s = h->stream;
        // per rank: Ctrl, partials [nb][ncols + 2], h1, h2, h3, T entry; mailbox block; PeerArgs
        const int PSp = (int)ncols + 2;
        const size_t mb = (peer_mailbox_bytes(P, kPeerPS) + 255) / 256 * 256;
        const size_t per = (sizeof(Ctrl) + 255) / 256 * 256 + ((size_t)nb * PSp + 3 * (size_t)PSp + 8) * sizeof(double);
        const size_t per_al = (per + 255) / 256 * 256;
        const size_t total = (size_t)P * (per_al + mb) + P * sizeof(PeerArgs) + cgs2_peer_emulate_grp_bytes(P) + 512;
        char *base = nullptr;
        ck(cudaMalloc(&base, total), "cudaMalloc");
        struct FreeB {
            char *p;
            ~FreeB() { cudaFree(p); }
        } fb{base};
        ck(cudaMemsetAsync(base, 0, total, s), "memset");
        std::vector<PeerEmuRank> ranks((size_t)P);
        std::vector<PeerArgs> pa((size_t)P);
        char *mbox0 = base + (size_t)P * per_al;
        PeerArgs *pa_dev = reinterpret_cast<PeerArgs *>(mbox0 + (size_t)P * mb);
        void *grp_dev = reinterpret_cast<char *>(pa_dev) + ((P * sizeof(PeerArgs) + 255) / 256 * 256);
        for (int q = 0; q < P; q++) {
            char *r = base + (size_t)q * per_al;
            Ctrl *ctrl = reinterpret_cast<Ctrl *>(r);
            double *d = reinterpret_cast<double *>(r + (sizeof(Ctrl) + 255) / 256 * 256);
            PeerEmuRank &e = ranks[q];
            e.N = row0[q + 1] - row0[q];
            e.Q = ncols > 0 ? Q + row0[q] : nullptr;
            e.ldq = ncols > 0 ? ldq : 2;
            e.w = w + row0[q];
            e.fs = FusedScratch{d, d + (size_t)nb * PSp, d + (size_t)nb * PSp + PSp, d + (size_t)nb * PSp + 2 * PSp,
                                ctrl->gflags, 16u, nullptr};
            e.ctrl = ctrl;
            e.t_entry = d + (size_t)nb * PSp + 3 * PSp;
            e.peer = pa_dev + q;
            PeerArgs &a = pa[q];
            a.P = P;
            a.rank = q;
            a.PS = kPeerPS;
            a.expect = (unsigned)(P * nb);
            char *mq = mbox0 + (size_t)q * mb;
            a.ctr = reinterpret_cast<unsigned int *>(mq);
            a.seq = reinterpret_cast<unsigned int *>(mq) + 2;
            a.mbox = reinterpret_cast<double *>(mq + kPeerHdrBytes);
            for (int z = 0; z < P; z++) {
                char *mz = mbox0 + (size_t)z * mb;
                a.ctr_peer[z] = reinterpret_cast<unsigned int *>(mz);
                a.mbox_peer[z] = reinterpret_cast<double *>(mz + kPeerHdrBytes);
            }
        }
        ck(cudaMemcpyAsync(pa_dev, pa.data(), P * sizeof(PeerArgs), cudaMemcpyHostToDevice, s), "H2D");
        if (!cgs2_peer_emulate(P, (int)ncols, ranks.data(), nb, grp_dev, s))
            throw SvdscError(SVDSC_ECUDA, "emulated multi-rank CGS2 launch failed");
        bool lost = false;
        for (int q = 0; q < P; q++) {
            Ctrl c;
            ck(cudaMemcpyAsync(&c, ranks[q].ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaMemcpyAsync(beta_out + q, ranks[q].t_entry, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaStreamSynchronize(s), "sync");
            lost = lost || (c.abort && c.abort_kind == 2);
        }
        ck(cudaGetLastError(), "cgs2 peer emulate");
        if (lost) throw CommError(SVDSC_ENCCL, "emulated peer exchange timed out");
    });
}

svdsc_status svdsc_op_small_svd(svdsc_handle *h, int32_t p, const double *Tm, double *U, double *S, double *V,
                                int32_t *sweeps) {
    if (!h) return SVDSC_EINVAL;
    svdsc_status ret = SVDSC_OK;
    svdsc_status st = guarded(h, [&] {
        einval(p < 1 || p > 1023 || !Tm || !U || !S || !V, "bad arguments");
        OpScratch sc = op_scratch(h, 0, p);
        cudaStream_t s = h->stream;
        small_svd(p, Tm, p, sc.W, sc.Vw, U, S, V, p, sc.ctrl, nullptr, sc.tlog, s);
        Ctrl c;
        ck(cudaMemcpyAsync(&c, sc.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
        ck(cudaGetLastError(), "small_svd");
        if (sweeps) *sweeps = c.svd_sweeps;
        if (c.svd_status != 0) ret = SVDSC_ESVD_NOCONV;
    });
    return st != SVDSC_OK ? st : ret;
}

svdsc_status svdsc_op_recombine(svdsc_handle *h, int64_t N, int32_t t, int32_t k, const double *Q, int64_t ldq,
                                const double *W, int32_t ldw, double *Qout, int64_t ldo) {
    if (!h) return SVDSC_EINVAL;
    return guarded(h, [&] {
        einval(N < 1 || t < 1 || t > 1023 || k < 1 || k > t || !Q || !W || !Qout || ldq < N || ldw < t || ldo < N,
               "bad arguments");
        recombine(N, t, k, Q, ldq, W, ldw, Qout, ldo, h->nsm, h->stream);
        ck(cudaGetLastError(), "recombine");
    });
}

svdsc_status svdsc_profile_enable(svdsc_handle *h, int enable) {
    if (!h) return SVDSC_EINVAL;
    cudaStreamSynchronize(h->stream);
    h->prof.harvest();
    h->prof.on = enable != 0;
    h->prof.mask = enable < 0 ? (unsigned)(-enable) : 0xffffffffu;
    for (int i = 0; i < SVDSC_PROF_FAMILIES; i++) {
        h->prof.ms[i] = 0.0;
        h->prof.calls[i] = 0;
    }
    return SVDSC_OK;
}

svdsc_status svdsc_profile_read(const svdsc_handle *h, double *ms, int64_t *calls) {
    if (!h || !ms || !calls) return SVDSC_EINVAL;
    for (int i = 0; i < SVDSC_PROF_FAMILIES; i++) {
        ms[i] = h->prof.ms[i];
        calls[i] = h->prof.calls[i];
    }
    return SVDSC_OK;
}

svdsc_status svdsc_comm_unique_id(unsigned char id[128]) {
    if (!id) return SVDSC_EINVAL;
    return guarded(nullptr, [&] { comm_nccl_unique_id(id); });
}

svdsc_status svdsc_comm_init(svdsc_handle *h, int nranks, int rank, const unsigned char id[128]) {
    if (!h || !id || nranks < 1 || rank < 0 || rank >= nranks) return SVDSC_EINVAL;
    return guarded(h, [&] {
        delete h->comm;
        h->comm = nullptr;
        h->nranks = 1;
        h->rank = 0;
        // (a one-rank communicator is created too: the solver runs its single-GPU
        // path, svdsc_comm_check exercises the collectives)
        h->comm = comm_nccl_create(id, nranks, rank);
        h->nranks = nranks;
        h->rank = rank;
    });
}

svdsc_status svdsc_comm_check(svdsc_handle *h) {
    if (!h) return SVDSC_EINVAL;
    return guarded(h, [&] {
        einval(!h->comm, "no communicator (svdsc_comm_init / svdsc_comm_init_group first)");
        Comm *c = h->comm;
        const int P = c->nranks, r = c->rank;
        constexpr int E = 5, A = 7;
        cudaStream_t s = h->stream;
        std::vector<double> hb((size_t)2 * E + 2 * (size_t)E * P + A);
        double *ag_in = hb.data(), *ag_out = ag_in + E, *rs_in = ag_out + (size_t)E * P, *rs_out = rs_in + (size_t)E * P,
               *ar = rs_out + E;
        for (int i = 0; i < E; i++) ag_in[i] = r * 10 + i;
        for (int i = 0; i < E * P; i++) rs_in[i] = (double)(r + 1) * (i + 1);
        for (int i = 0; i < A; i++) ar[i] = r + 1 + i;
        double *d = nullptr;
        ck(cudaMalloc(&d, hb.size() * sizeof(double)), "cudaMalloc");
        struct Free {
            double *p;
            ~Free() { cudaFree(p); }
        } fr{d};
        ck(cudaMemcpyAsync(d, hb.data(), hb.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
        const size_t o_ago = E, o_rsi = o_ago + (size_t)E * P, o_rso = o_rsi + (size_t)E * P, o_ar = o_rso + E;
        c->allgather(d, d + o_ago, E, s);
        c->reduce_scatter_sum(d + o_rsi, d + o_rso, E, s);
        c->allreduce_sum(d + o_ar, A, s);
        ck(cudaMemcpyAsync(hb.data(), d, hb.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
        const int mn = c->allreduce_min_int(r + 3, s);
        const double tri = 0.5 * P * (P + 1);
        bool ok = mn == 3;
        for (int q = 0; q < P; q++)
            for (int i = 0; i < E; i++) ok = ok && ag_out[q * E + i] == q * 10 + i;
        for (int i = 0; i < E; i++) ok = ok && rs_out[i] == tri * (r * E + i + 1);
        for (int i = 0; i < A; i++) ok = ok && ar[i] == tri + (double)P * i;
        if (!ok) throw CommError(SVDSC_ENCCL, "communicator check: collective results differ from the expected sums");
        // the peer mailboxes (NCCL backend): one in-kernel exchange
        c->peer_reset(s);
        (void)c->allreduce_min_int(0, s);  // every rank has reset before any arrival
        const PeerArgs *pa = c->peer_setup(h->nsm, s);
        if (pa) {
            constexpr int X = 9;
            OpScratch sc = op_scratch(h, 0, 1);
            double *dx = nullptr;
            ck(cudaMalloc(&dx, X * sizeof(double)), "cudaMalloc");
            Free fx{dx};
            ck(cudaMemsetAsync(sc.ctrl, 0, sizeof(Ctrl), s), "memset");
            peer_check(pa, X, dx, sc.ctrl, s);
            double hx[X];
            Ctrl cc;
            ck(cudaMemcpyAsync(hx, dx, sizeof(hx), cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaMemcpyAsync(&cc, sc.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s), "D2H");
            ck(cudaStreamSynchronize(s), "sync");
            ck(cudaGetLastError(), "peer_check");
            bool pok = cc.abort_kind != 2;
            for (int j = 0; j < X; j++) pok = pok && hx[j] == tri * (j + 1);
            if (c->allreduce_min_int(pok ? 1 : 0, s) != 1)
                throw CommError(SVDSC_ENCCL, "communicator check: peer-mailbox exchange failed");
        }
    });
}

svdsc_status svdsc_group_create(int nranks, svdsc_group **g) {
    if (!g || nranks < 1 || nranks > 16) return SVDSC_EINVAL;
    *g = new svdsc_group{loopback_group_create(nranks), nranks};
    return SVDSC_OK;
}

void svdsc_group_destroy(svdsc_group *g) {
    if (!g) return;
    loopback_group_release(g->g);
    delete g;
}

svdsc_status svdsc_comm_init_group(svdsc_handle *h, svdsc_group *g, int rank) {
    if (!h || !g || !g->g) return SVDSC_EINVAL;
    return guarded(h, [&] {
        einval(rank < 0 || rank >= g->nranks(), "rank out of range");
        delete h->comm;
        h->comm = nullptr;
        h->nranks = 1;
        h->rank = 0;
        h->comm = comm_loopback_create(g->g, rank);
        h->nranks = g->nranks();
        h->rank = rank;
    });
}

svdsc_status svdsc_set_policy(svdsc_handle *h, int32_t key, int32_t value) {
    if (!h) return SVDSC_EINVAL;
    const int maxv[4] = {2, 7, 3, 1};
    if (key < 0 || key > 3 || value < 0 || value > maxv[key]) {
        h->err = "svdsc_set_policy: unknown key or value";
        return SVDSC_EINVAL;
    }
    if (key == SVDSC_POLICY_SPMV) h->policy.spmv = value;
    else if (key == SVDSC_POLICY_CGS2) h->policy.cgs2 = value;
    else if (key == SVDSC_POLICY_DEFER) h->policy.defer = value;
    else h->policy.small_svd = value;
    return SVDSC_OK;
}

svdsc_status svdsc_partition_rows(int64_t m, const int64_t *row_ptr, int64_t basis_cols, int nparts, int64_t *bounds) {
    if (m < 0 || !row_ptr || nparts < 1 || !bounds || basis_cols < 0) return SVDSC_EINVAL;
    // cost(r) = 24 nnz_r + 24 basis_cols  (A read twice at 12 B/nnz; three U sweeps)
    const long double total = 24.0L * (long double)row_ptr[m] + 24.0L * basis_cols * (long double)m;
    bounds[0] = 0;
    int64_t r = 0;
    long double acc = 0.0L;
    for (int q = 1; q < nparts; q++) {
        const long double target = total * q / nparts;
        while (r < m) {
            const long double c = 24.0L * (row_ptr[r + 1] - row_ptr[r]) + 24.0L * basis_cols;
            if (acc + c / 2 > target) break;
            acc += c;
            r++;
        }
        bounds[q] = r;
    }
    bounds[nparts] = m;
    for (int q = 1; q <= nparts; q++)
        if (bounds[q] < bounds[q - 1]) return SVDSC_EINVAL;
    return SVDSC_OK;
}

}  // extern "C"
