// cgs_fused.cu -- one persistent kernel per re-orthogonalization (single GPU):
// the two classical Gram-Schmidt passes of PAPER.md:121 (reading Q1), the norm
// that gives alpha/beta (Alg. 1 lines 6 and 8) and the normalization, with the
// three global reductions done by a grid barrier instead of kernel boundaries.
//
// Each CTA owns a contiguous block of rows for the whole kernel:
//   phase A  partial h1 = Q_b^T w_b                       (read Q once)
//   phase B  w' = w - Q h1;  partial h2 = Q_b^T w'_b, ||w'_b||^2
//            (a row tile of Q is staged in shared memory and used twice)
//   phase C  w'' = w' - Q h2 (read Q once); beta from the Pythagorean identity
//            ||w''||^2 = ||w'||^2 - ||h2||^2 (Q orthonormal) when the second
//            pass removed less than half of ||w'||^2, else an explicit extra
//            reduction; breakdown test (reading Q7); v = w'' / beta.
// If the CTA's rows of Q fit in shared memory (small bases, e.g. BASELINE
// configs 1-2) Q is read from HBM once instead of three times.
// Reductions over CTAs: partials [block][column], then CTA b reduces columns
// b, b + nb, ... in a fixed tree order (deterministic), grid barrier, and
// every CTA reads the reduced vector.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace svdsc {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// fixed-order block sum, result broadcast to every thread
__device__ __forceinline__ double block_sum_all(double v, double *sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += sh[i];
    __syncthreads();
    return s;
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}


// Grid barrier over all CTAs of a cooperative launch, on a monotonic arrival
// counter: every CTA adds 1 (red.release, no return value) and polls until the
// counter reaches n x gridDim.x for the launch's n-th barrier (1.2 us per
// barrier on B200 vs 2.4 us for a returning atomicAdd + generation flag,
// tools/barrier_bench.cu).  `v` = epoch + n with epoch a per-launch multiple of
// 16 (n < 16); launch epoch/16 owns counter slot (epoch/16) % 512, which the
// previous launch on the stream zeroed (grid_prepare) and the per-solve /
// per-op Ctrl memset zeroes initially.
constexpr int kBarSlots = 512;
__device__ __forceinline__ void red_release_add(unsigned int *p, unsigned int v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void grid_sync(unsigned int *flags, unsigned int v) {
    unsigned int *ctr = flags + 2 + ((v >> 4) & (kBarSlots - 1));
    const unsigned int target = (v & 15u) * gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        red_release_add(ctr, 1u);
        while (ld_acquire(ctr) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}
// zero the barrier slot of the NEXT launch (stream order makes this safe)
__device__ __forceinline__ void grid_prepare(unsigned int *flags, unsigned int epoch) {
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[2 + (((epoch >> 4) + 1) & (kBarSlots - 1))] = 0u;
}
// the same over a group of nb CTAs (bid = index in the group): the grid of one
// rank in an emulated multi-rank launch, else the whole grid
__device__ __forceinline__ void grid_sync_n(unsigned int *flags, unsigned int v, int nb) {
    unsigned int *ctr = flags + 2 + ((v >> 4) & (kBarSlots - 1));
    const unsigned int target = (v & 15u) * (unsigned)nb;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        red_release_add(ctr, 1u);
        while (ld_acquire(ctr) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_prepare_n(unsigned int *flags, unsigned int epoch, int bid) {
    if (bid == 0 && threadIdx.x == 0) flags[2 + (((epoch >> 4) + 1) & (kBarSlots - 1))] = 0u;
}
// system scope (another GPU's memory over NVLink): peer mailbox protocol
__device__ __forceinline__ void red_release_sys_add(unsigned int *p, unsigned int v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// a peer that never arrives (a dead rank) ends the wait after ~2^34 cycles
// (~9 s) with ctrl->abort_kind = 2 instead of hanging the job
constexpr long long kPeerTimeoutCycles = 1LL << 34;

constexpr int kTile = 16;

__device__ __forceinline__ double butterfly16(double (&acc)[kTile], int lane) {
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
        const bool hi = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < off; q++) {
            double send = hi ? acc[q] : acc[q + off];
            double keep = hi ? acc[q + off] : acc[q];
            acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 16);
}

struct Args {
    int64_t N;
    int ncols;
    const double *Q;
    int64_t ldq;
    double *w;
    double *partial;  // [nb][PS]
    int PS;
    double *h1, *h2, *h3;
    unsigned int *flags;  // grid-barrier flags (one per CTA)
    unsigned int epoch;   // base epoch of this launch
    Ctrl *ctrl;
    double *t_entry;
    int check;
    const double *pre_h;  // optional w -= Q pre_h before the passes (Alg. 2 step 10)
    int rpb;              // rows per CTA
    int RT;               // row tile of phase B (streaming mode)
    int wsmem;            // keep the CTA's w rows in shared memory
    PreReduce pre;        // pending split-K reduction of w (pre.partial != NULL)
    const int *gate;      // partial re-orthogonalization gate (FusedScratch::gate)
    int gate_want;
};

// out[j] = sum_b partial[b][j] for the columns owned by this CTA
__device__ void reduce_cols(const Args &a, int ncols_tot, double *out, double *) {
    const int nb = gridDim.x, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int tw = gridDim.x * nw;
    for (int j = blockIdx.x * nw + (threadIdx.x >> 5); j < ncols_tot; j += tw) {
        double s = 0.0;
        for (int t = lane; t < nb; t += 32) s += __ldcg(a.partial + (int64_t)t * a.PS + j);
        s = warp_sum(s);
        if (lane == 0) out[j] = s;
    }
}

template <bool QS>
__device__ __forceinline__ double qval(const Args &a, const double *qsh, int ldqs, int64_t r0, int i, int j) {
    if (QS) return qsh[j * ldqs + i];
    return __ldg(a.Q + r0 + i + (int64_t)j * a.ldq);
}

template <bool QS>
__global__ void __launch_bounds__(256) k_cgs2_fused(Args a) {
    grid_prepare(a.flags, a.epoch);
    if (*(volatile int *)&a.ctrl->abort) return;  // uniform over the grid
    if (a.gate && *(volatile const int *)a.gate != a.gate_want) return;  // PRO gate, uniform
    unsigned int nbar = 0;
    extern __shared__ double sm[];
    __shared__ double sh[32];
    __shared__ double sred[8][kTile];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ncols = a.ncols;
    const int64_t r0 = (int64_t)blockIdx.x * a.rpb;
    const int nr = (int)max((int64_t)0, min((int64_t)a.rpb, a.N - r0));
    const int ldqs = a.rpb + 1;
    // shared layout
    double *hs = sm;                         // ncols (+1)
    double *wsh = hs + ncols + 2;            // rpb (if wsmem)
    double *qsh = wsh + (a.wsmem ? a.rpb : 0);  // QS: ncols x (rpb+1); else tile ncols x (RT+1)
    const int LDT = a.RT + 1;
    double *part = qsh + (QS ? (int64_t)ncols * ldqs : (int64_t)ncols * LDT);  // 256 (QS: row-dot scratch)
    double *wpt = part + 256;                               // RT
    double *wv = a.wsmem ? wsh : (a.w + r0);  // generic pointer to this CTA's rows of w

    if (a.wsmem)
        for (int i = tid; i < nr; i += blockDim.x) {
            if (a.pre.partial) {  // finish the dense product (k_split_reduce order: bitwise equal)
                double sacc = 0.0;
                for (int q = 0; q < a.pre.splits; q++) sacc += a.pre.partial[q * a.N + r0 + i];
                if (a.pre.yprev) sacc -= *a.pre.c_dev * a.pre.yprev[r0 + i];
                wsh[i] = sacc;
            } else {
                wsh[i] = a.w[r0 + i];
            }
        }
    if (QS) {  // the CTA's rows of Q, all copies in flight at once (cp.async, 8 B each)
        for (int j = wid; j < ncols; j += 8)
            for (int i = lane; i < nr; i += 32) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(qsh + j * ldqs + i);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(a.Q + r0 + i + (int64_t)j * a.ldq));
            }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (a.pre_h) {  // w -= Q pre_h (restart, Eq. (7))
        for (int j = tid; j < ncols; j += blockDim.x) hs[j] = a.pre_h[j];
        __syncthreads();
        for (int i = tid; i < nr; i += blockDim.x) {
            double s = 0.0;
            for (int j = 0; j < ncols; j++) s = fma(qval<QS>(a, qsh, ldqs, r0, i, j), hs[j], s);
            wv[i] -= s;
        }
        __syncthreads();
    }

    // QS helpers.  Column dots: one thread per column, four interleaved chains
    // over the CTA's rows (ldqs odd: the 32 columns of a warp hit 32 banks).
    auto qs_coldots = [&](const double *v) {
        for (int j = tid; j < ncols; j += blockDim.x) {
            const double *qj = qsh + j * ldqs;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int i = 0;
            for (; i + 4 <= nr; i += 4) {
                s0 = fma(qj[i], v[i], s0);
                s1 = fma(qj[i + 1], v[i + 1], s1);
                s2 = fma(qj[i + 2], v[i + 2], s2);
                s3 = fma(qj[i + 3], v[i + 3], s3);
            }
            for (; i < nr; i++) s0 = fma(qj[i], v[i], s0);
            a.partial[(int64_t)blockIdx.x * a.PS + j] = (s0 + s1) + (s2 + s3);
        }
    };
    // Row dots Q_b h: thread (row i, column group g) sums columns g, g + G, ...;
    // the G partials of a row are combined in fixed order.  Result in rdot[i].
    double *rdot = part;  // >= max(256, rpb) doubles of scratch (part region)
    auto qs_rowdots = [&](const double *h) {
        const int G = (int)blockDim.x / max(nr, 1);
        if (G <= 1) {  // at least as many rows as threads: one thread per row
            for (int i = tid; i < nr; i += blockDim.x) {
                double s0 = 0.0, s1 = 0.0;
                int j = 0;
                for (; j + 1 < ncols; j += 2) {
                    s0 = fma(qsh[j * ldqs + i], h[j], s0);
                    s1 = fma(qsh[(j + 1) * ldqs + i], h[j + 1], s1);
                }
                if (j < ncols) s0 = fma(qsh[j * ldqs + i], h[j], s0);
                rdot[i] = s0 + s1;
            }
            __syncthreads();
            return;
        }
        const int i = tid % max(nr, 1), g = tid / max(nr, 1);
        double s0 = 0.0, s1 = 0.0;
        if (g < G && i < nr) {
            int j = g;
            for (; j + G < ncols; j += 2 * G) {
                s0 = fma(qsh[j * ldqs + i], h[j], s0);
                s1 = fma(qsh[(j + G) * ldqs + i], h[j + G], s1);
            }
            if (j < ncols) s0 = fma(qsh[j * ldqs + i], h[j], s0);
        }
        __syncthreads();
        if (g < G && i < nr) rdot[g * nr + i] = s0 + s1;
        __syncthreads();
        if (tid < nr) {
            double t = 0.0;
            for (int q = 0; q < G; q++) t += rdot[q * nr + tid];
            rdot[tid] = t;  // (G partials of row tid read above by this thread only)
        }
        __syncthreads();
    };

    double nrm_wp = 0.0;  // ||w'||^2 partial (thread-local)
    if (ncols > 0) {
        // ---------------- phase A: partial h1 ----------------
        if (QS) {
            qs_coldots(wv);
        } else {
            for (int j0 = 0; j0 < ncols; j0 += kTile) {
                const int nc = min(kTile, ncols - j0);
                double acc[kTile];
#pragma unroll
                for (int q = 0; q < kTile; q++) acc[q] = 0.0;
                for (int i = tid; i < nr; i += blockDim.x) {
                    const double wr = wv[i];
                    const double *qp = a.Q + r0 + i + (int64_t)j0 * a.ldq;
#pragma unroll
                    for (int q = 0; q < kTile; q++)
                        if (q < nc) acc[q] = fma(__ldg(qp + (int64_t)q * a.ldq), wr, acc[q]);
                }
                const double v = butterfly16(acc, lane);
                if (lane < kTile) sred[wid][lane] = v;
                __syncthreads();
                if (tid < nc) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < 8; q++) s += sred[q][tid];
                    a.partial[(int64_t)blockIdx.x * a.PS + j0 + tid] = s;
                }
                __syncthreads();
            }
        }
        grid_sync(a.flags, a.epoch + (++nbar));
        reduce_cols(a, ncols, a.h1, sh);
        grid_sync(a.flags, a.epoch + (++nbar));
        for (int j = tid; j < ncols; j += blockDim.x) hs[j] = __ldcg(a.h1 + j);
        __syncthreads();

        // ---------------- phase B: w' = w - Q h1, partial h2, ||w'||^2 ----------------
        if (QS) {
            qs_rowdots(hs);
            for (int i = tid; i < nr; i += blockDim.x) {
                const double v = wv[i] - rdot[i];
                wv[i] = v;
                nrm_wp = fma(v, v, nrm_wp);
            }
            __syncthreads();
            qs_coldots(wv);
        } else {
            const int RT = a.RT, P = blockDim.x / RT;
            const int rr = tid % RT, pp = tid / RT;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int t0 = 0; t0 < nr; t0 += RT) {
                const int tn = min(RT, nr - t0);
                for (int idx = tid; idx < ncols * RT; idx += blockDim.x) {
                    const int j = idx / RT, q = idx - j * RT;
                    qsh[j * LDT + q] = (q < tn) ? __ldg(a.Q + r0 + t0 + q + (int64_t)j * a.ldq) : 0.0;
                }
                __syncthreads();
                double s = 0.0;
                for (int j = pp; j < ncols; j += P) s = fma(qsh[j * LDT + rr], hs[j], s);
                part[pp * RT + rr] = s;
                __syncthreads();
                if (tid < RT) {
                    double ts = 0.0;
                    for (int q = 0; q < P; q++) ts += part[q * RT + tid];
                    double v = 0.0;
                    if (tid < tn) {
                        v = wv[t0 + tid] - ts;
                        wv[t0 + tid] = v;
                        nrm_wp = fma(v, v, nrm_wp);
                    }
                    wpt[tid] = v;
                }
                __syncthreads();
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int j = tid + 256 * q;
                    if (j < ncols) {
                        double x = acc[q];
                        const double *tj = qsh + j * LDT;
                        for (int k = 0; k < RT; k++) x = fma(tj[k], wpt[k], x);
                        acc[q] = x;
                    }
                }
                __syncthreads();
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int j = tid + 256 * q;
                if (j < ncols) a.partial[(int64_t)blockIdx.x * a.PS + j] = acc[q];
            }
        }
        const double bn = block_sum_all(nrm_wp, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS + ncols] = bn;
        grid_sync(a.flags, a.epoch + (++nbar));
        reduce_cols(a, ncols + 1, a.h2, sh);
        grid_sync(a.flags, a.epoch + (++nbar));
        for (int j = tid; j <= ncols; j += blockDim.x) hs[j] = __ldcg(a.h2 + j);
        __syncthreads();
    } else {
        // plain norm: ||w||^2 into hs[0] (ncols == 0)
        for (int i = tid; i < nr; i += blockDim.x) nrm_wp = fma(wv[i], wv[i], nrm_wp);
        const double bn = block_sum_all(nrm_wp, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS] = bn;
        grid_sync(a.flags, a.epoch + (++nbar));
        reduce_cols(a, 1, a.h2, sh);
        grid_sync(a.flags, a.epoch + (++nbar));
        if (tid == 0) hs[0] = __ldcg(a.h2);
        __syncthreads();
    }

    // ---------------- phase C: w'' = w' - Q h2, beta, breakdown, normalize ----------------
    const double nrmp = hs[ncols];
    double hh = 0.0;
    for (int j = tid; j < ncols; j += blockDim.x) hh = fma(hs[j], hs[j], hh);
    hh = block_sum_all(hh, sh);
    double beta2 = nrmp - hh;
    const bool pyth = beta2 > 0.5 * nrmp;
    double nrm2 = 0.0;
    if (ncols > 0) {
        if (QS) {
            qs_rowdots(hs);
            for (int i = tid; i < nr; i += blockDim.x) {
                const double v = wv[i] - rdot[i];
                wv[i] = v;
                nrm2 = fma(v, v, nrm2);
            }
        } else {
            for (int i = tid; i < nr; i += blockDim.x) {
                double s = 0.0;
#pragma unroll 8
                for (int j = 0; j < ncols; j++) s = fma(qval<QS>(a, qsh, ldqs, r0, i, j), hs[j], s);
                const double v = wv[i] - s;
                wv[i] = v;
                nrm2 = fma(v, v, nrm2);
            }
        }
    }
    __syncthreads();
    if (!pyth) {  // explicit norm (uniform branch: every CTA sees the same hs)
        const double bn = block_sum_all(nrm2, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS] = bn;
        grid_sync(a.flags, a.epoch + (++nbar));
        reduce_cols(a, 1, a.h3, sh);
        grid_sync(a.flags, a.epoch + (++nbar));
        beta2 = __ldcg(a.h3);
    }
    const double beta = sqrt(fmax(beta2, 0.0));
    const double amax = a.ctrl->amax[a.check & 1];
    const bool bd = !(beta > 1e-14 * fmax(amax, 1.0));
    if (blockIdx.x == 0 && tid == 0) {
        if (bd) {
            *a.t_entry = 0.0;
            a.ctrl->amax[(a.check + 1) & 1] = amax;
            a.ctrl->abort_check = a.check;
            __threadfence();
            a.ctrl->abort = 1;
        } else {
            *a.t_entry = beta;
            a.ctrl->amax[(a.check + 1) & 1] = fmax(amax, beta);
        }
    }
    if (!bd)
        for (int i = tid; i < nr; i += blockDim.x) a.w[r0 + i] = wv[i] / beta;
}

// ---------------------------------------------------------------------------
// Streaming variant for tall bases (Q does not fit on chip): each CTA owns a
// contiguous range of rows and streams it through shared memory in row tiles
// of RT rows x ncols, loaded with cp.async (16-byte chunks, double-buffered,
// zero-filled tails) into an XOR-swizzled layout so that both access patterns
// -- lane per row (row updates) and thread per column (column dots) -- are
// bank-conflict free.  Three sweeps over Q (the CGS2 minimum), one grid
// barrier pair per global reduction.
struct SArgs {
    int64_t N;
    int ncols;
    const double *Q;
    int64_t ldq;
    double *w;
    double *partial;
    int PS;
    double *h1, *h2, *h3;
    unsigned int *flags;  // grid-barrier flags (one per CTA)
    unsigned int epoch;   // base epoch of this launch
    Ctrl *ctrl;
    double *t_entry;
    int check;
    const double *pre_h;
    int64_t rpb;  // rows per CTA, multiple of RT
    int snake;    // stream2 sweep direction: 1 alternate (default), 2 only with a 2-stage ring
    // stream2 only: 0 = the whole CGS2 in one launch (single GPU); 1 / 2 / 3 =
    // one phase of it (multi-GPU: the host all-reduces h1, then [h2; ||w'||^2],
    // across the ranks between the launches): 1 = [pre_h sweep] + h1 (CTA-reduced
    // into h1), 2 = w' and h2, ||w'||^2 (into h2[0..ncols]), 3 = w'', beta,
    // normalization -- where the explicit norm is needed (reading G1) phase 3
    // leaves w'' unnormalized and raises ctrl->abort with abort_kind = 1
    int phase;
    const int *gate;      // partial re-orthogonalization gate (FusedScratch::gate)
    int gate_want;
    // peer instantiation (k_cgs2_stream2p, cgs2_peer): the rank's mailbox, whose
    // one-shot all-reduces replace the host all-reduces of the phased launches
    const PeerArgs *peer;
    // deferred second update (single GPU; internal.h DeferState): dst = this
    // side's state, qw = Q (writable: the pending column is formed in place),
    // xs = the next product's input, defer = leave this call's column pending
    DeferState *dst;
    double *qw;
    double *xs;
    int defer;
};

template <int RT>
struct Tiles {
    static constexpr int kCh = RT / 2;  // 16-byte chunks per column per tile
    __device__ static __forceinline__ int swz(int j, int c) { return j * RT + ((c ^ (j & (kCh - 1))) << 1); }
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src, int bytes) {
    const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


// issue the loads of one row tile (Q rows [r, r+nr) of all columns, and w rows).
// Thread t always moves chunk c = t % kCh of columns j = t / kCh + u (kSThr/kCh),
// so addresses advance by constant strides (no per-chunk index arithmetic).
template <int RT, int kSThr>
__device__ __forceinline__ void issue_tile(const SArgs &a, double *buf, double *wt, int64_t r, int nr) {
    constexpr int kCh = RT / 2;
    constexpr int CPI = kSThr / kCh;  // columns per iteration
    const int c = threadIdx.x % kCh, j0 = threadIdx.x / kCh;
    const double *src = a.Q + r + 2 * c + (int64_t)j0 * a.ldq;
    const int64_t sstep = (int64_t)CPI * a.ldq;
    double *dst = buf + j0 * RT + ((c ^ (j0 & (kCh - 1))) << 1);  // (j0 + CPI u) & (kCh-1) == j0 & (kCh-1)
    constexpr int dstep = CPI * RT;
    if (nr == RT) {
        for (int j = j0; j < a.ncols; j += CPI, src += sstep, dst += dstep) cp_async16(dst, src, 16);
    } else {
        const int bytes = min(16, max(0, (nr - 2 * c) * 8));
        for (int j = j0; j < a.ncols; j += CPI, src += sstep, dst += dstep) cp_async16(dst, bytes ? src : a.Q, bytes);
    }
    if (threadIdx.x < kCh) {
        const int bytes = min(16, max(0, (nr - 2 * c) * 8));
        cp_async16(wt + 2 * c, bytes ? a.w + r + 2 * c : a.w, bytes);
    }
    cp_commit();
}

// one warp per column (fixed lane-strided order + xor tree: deterministic);
// a block-wide reduction per column cost ~2 us per column (3 __syncthreads)
__device__ void sreduce_cols(const SArgs &a, int ncols_tot, double *out, int bid, int nb) {
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int tw = nb * nw;
    for (int j = bid * nw + (threadIdx.x >> 5); j < ncols_tot; j += tw) {
        double s = 0.0;
        for (int t = lane; t < nb; t += 32) s += __ldcg(a.partial + (int64_t)t * a.PS + j);
        s = warp_sum(s);
        if (lane == 0) out[j] = s;
    }
}

// ---------------------------------------------------------------------------
// Streaming CGS2, register-blocked variant: warp w owns rows w, w+16, ... of
// every row tile, lane q owns columns q, q+32, ..., q+32(M-1).  Column dots
// (h1, h2) accumulate in registers across all tiles and are combined across
// warps once per phase; row dots (w', w'') are one warp reduction per row.
// The tile body has no __syncthreads (only the cp.async ring's two per tile).
// bid / nb: this CTA's index among the rank's CTAs and their number (the grid,
// except in an emulated multi-rank launch).  PEER: the global reductions are
// completed across the ranks inside the kernel (PeerArgs, internal.h).
// RT = 32 instances with M >= 6 keep the shared-memory tile 32 M columns wide
// (columns past ncols zero): the sweeps then read the lane's columns
// unpredicated.  The M = 2, 4 instances measured slower padded (r02p launch
// list: 876 vs 786 us, 1194 vs 1095 us; <32,4,4> spills once unpredicated) and
// the RT = 16 instances (up to 1024 columns) keep the tight layout
template <int RT, int M>
__host__ __device__ constexpr bool stream2_pad() { return RT == 32 && M >= 6; }
template <int RT, int M>
__host__ __device__ inline int stream2_tcols(int ncols) { return stream2_pad<RT, M>() ? 32 * M : ncols; }

template <int RT, int NS, int M, bool PEER>
__device__ __forceinline__ void cgs2_stream2_body(const SArgs &a, const int bid, const int nb) {
    constexpr int kSThr = 512, NW = 16, RPW = RT / NW, kCh = RT / 2;
    grid_prepare_n(a.flags, a.epoch, bid);
    if (*(volatile int *)&a.ctrl->abort) return;
    if (!PEER && a.gate && *(volatile const int *)a.gate != a.gate_want) return;  // PRO gate, uniform
    unsigned int nbar = 0;
    extern __shared__ __align__(16) double smem_s[];
    __shared__ double sh[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ncols = a.ncols;
    constexpr bool kPad = stream2_pad<RT, M>();
    const int tile_d = stream2_tcols<RT, M>(ncols) * RT;
    double *buf = smem_s;               // NS x tcols x RT (swizzled)
    double *wt = buf + NS * tile_d;     // NS x RT
    // columns [ncols, 32 M) of every stage: zero once per launch (the ring's
    // copies write columns < ncols only, the reduction scratch `red` stays
    // below 16 (ncols + 1) <= 32 ncols doubles of stage 0), so every sweep
    // reads the lane's M columns without a predicate (0 x 0 terms)
    if constexpr (kPad) {
        const int pad = (32 * M - ncols) * RT;
        for (int p = 0; p < NS; p++)
            for (int i = tid; i < pad; i += kSThr) buf[p * tile_d + ncols * RT + i] = 0.0;
    }
    auto colok = [&](int m) { return kPad || lane + 32 * m < ncols; };
    // NW x ncols cross-warp column sums: aliases the ring, which is idle when
    // a phase flushes (its last tile consumed, the next prefetch not issued)
    double *red = buf;
    const int64_t rb = (int64_t)bid * a.rpb;
    const int64_t re = min(a.N, rb + a.rpb);
    const int ntiles = rb < re ? (int)((re - rb + RT - 1) / RT) : 0;
    const int sw = lane & (kCh - 1);  // swizzle term of every column this lane owns

    // sweeps alternate direction (forward, backward, ...): each sweep starts on
    // the tiles the previous one read last, which are still in L2
    // (measured gain for the 2-stage ring, loss for the 3-stage one: snake only
    // where it wins, SVDSC_SNAKE=0/1/2 = never/always/2-stage)
    int sweep_no = 0;
    const bool snake = a.snake == 1 || (a.snake == 2 && NS == 2);
    auto tile_of = [&](int k) { return (snake && (sweep_no & 1)) ? ntiles - 1 - k : k; };
    // prologue: the first NS-1 tiles of a phase (issued early, e.g. before the
    // grid barrier of the previous reduction, so the ramp-up hides behind it)
    auto prefetch = [&]() {
#pragma unroll
        for (int p = 0; p < NS - 1; p++) {
            if (p < ntiles) {
                const int64_t r1 = rb + (int64_t)tile_of(p) * RT;
                issue_tile<RT, kSThr>(a, buf + p * tile_d, wt + p * RT, r1, (int)min((int64_t)RT, re - r1));
            } else {
                cp_commit();
            }
        }
    };
    bool prefetched = false;
    auto issue_next = [&](int kn) {
        if (kn < ntiles) {
            const int64_t r1 = rb + (int64_t)tile_of(kn) * RT;
            issue_tile<RT, kSThr>(a, buf + (kn % NS) * tile_d, wt + (kn % NS) * RT, r1,
                                  (int)min((int64_t)RT, re - r1));
        } else {
            cp_commit();
        }
    };
    auto run_tiles = [&](auto &&body) {
        if (ntiles == 0) return;
        if (!prefetched) prefetch();
        prefetched = false;
        for (int k = 0; k < ntiles; k++) {
            if constexpr (NS >= 3) {
                // one barrier per tile: it publishes tile k AND retires tile k-1,
                // whose slot the next tile is then issued into (measured: 140.2
                // vs 142.9 us per call at config 3; with two stages the issue
                // must stay ahead of the wait, below)
                cp_wait<NS - 2>();
                __syncthreads();
                issue_next(k + NS - 1);
                body(tile_of(k), buf + (k % NS) * tile_d, wt + (k % NS) * RT);
                continue;
            }
            issue_next(k + NS - 1);
            cp_wait<NS - 1>();
            __syncthreads();
            body(tile_of(k), buf + (k % NS) * tile_d, wt + (k % NS) * RT);
            __syncthreads();
        }
        cp_wait<0>();
        __syncthreads();  // the last tile is consumed before the ring is reused (red aliases it)
        sweep_no++;
    };
    // element (row rr, column lane + 32 m) of a tile
    auto tval = [&](const double *T, int rr, int m) -> double {
        return T[(lane + 32 * m) * RT + (((rr >> 1) ^ sw) << 1) + (rr & 1)];
    };
    // RPW == 2: the warp's rows are 2 wid and 2 wid + 1, one 16-byte chunk of
    // the swizzled tile per column -- both with one shared load
    auto tpair = [&](const double *T, int m) -> double2 {
        return *reinterpret_cast<const double2 *>(T + (lane + 32 * m) * RT + ((wid ^ sw) << 1));
    };
    // sums of the warp's RPW row partials.  RPW == 2 is a reduce-scatter: the
    // first level swaps the other row's partial across the half-warps, so both
    // rows take 5 shuffles instead of 10.  Afterwards p[q] is valid on lanes
    // [q * kHalf, (q + 1) * kHalf); row q is written by lane q * kHalf.
    static_assert(RPW == 1 || RPW == 2, "stream2 handles 1 or 2 rows per warp");
    constexpr int kHalf = 32 / RPW;
    auto reduce_rows = [&](double (&p)[RPW]) {
        if constexpr (RPW == 2) {
            const bool hi = lane & 16;
            double x = (hi ? p[1] : p[0]) + __shfl_xor_sync(0xffffffffu, hi ? p[0] : p[1], 16);
#pragma unroll
            for (int off = 8; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
            p[0] = x;
            p[1] = x;
        } else {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
        }
    };
    // the warp's RPW row dots with the lane's coefficients hreg
    auto rowdots = [&](const double *T, const double (&hreg)[M], double (&out)[RPW]) {
        if constexpr (RPW == 2) {
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int m = 0; m < M; m++) {
                if (colok(m)) {
                    const double2 t = tpair(T, m);
                    if (m & 1) {
                        a1 = fma(t.x, hreg[m], a1);
                        b1 = fma(t.y, hreg[m], b1);
                    } else {
                        a0 = fma(t.x, hreg[m], a0);
                        b0 = fma(t.y, hreg[m], b0);
                    }
                }
            }
            out[0] = a0 + a1;
            out[1] = b0 + b1;
        } else {
#pragma unroll
            for (int q = 0; q < RPW; q++) {
                const int rr = RPW * wid + q;
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int m = 0; m < M; m += 2) {
                    if (colok(m)) s0 = fma(tval(T, rr, m), hreg[m], s0);
                    if (m + 1 < M && lane + 32 * (m + 1) < ncols) s1 = fma(tval(T, rr, m + 1), hreg[m + 1], s1);
                }
                out[q] = s0 + s1;
            }
        }
        reduce_rows(out);
    };
    // the tile's values of the warp's rows into registers (zeros past ncols)
    // and their row dots with hreg: part[q] before the cross-lane reduction
    auto load_tile_rows = [&](const double *T, const double (&hreg)[M], double (&tv)[RPW][M], double (&part)[RPW]) {
        if constexpr (RPW == 2) {
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int m = 0; m < M; m++) {
                double2 t = make_double2(0.0, 0.0);
                if (colok(m)) t = tpair(T, m);
                tv[0][m] = t.x;
                tv[1][m] = t.y;
                if (m & 1) {
                    a1 = fma(t.x, hreg[m], a1);
                    b1 = fma(t.y, hreg[m], b1);
                } else {
                    a0 = fma(t.x, hreg[m], a0);
                    b0 = fma(t.y, hreg[m], b0);
                }
            }
            part[0] = a0 + a1;
            part[1] = b0 + b1;
        } else {
#pragma unroll
            for (int q = 0; q < RPW; q++) {
                const int rr = RPW * wid + q;
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int m = 0; m < M; m++) {
                    tv[q][m] = colok(m) ? tval(T, rr, m) : 0.0;
                    if (m & 1) s1 = fma(tv[q][m], hreg[m], s1);
                    else s0 = fma(tv[q][m], hreg[m], s0);
                }
                part[q] = s0 + s1;
            }
        }
    };
    // every lane needs both rows' values (phase B's column accumulation)
    auto allrows = [&](double (&p)[RPW]) {
        if constexpr (RPW == 2) {
            const double other = __shfl_xor_sync(0xffffffffu, p[0], 16);
            if (lane & 16) p[0] = other;
            else p[1] = other;
        }
    };
    // cross-warp column sums of acc -> partial[block][j]; with a norm, the
    // thread partials nrm (summed per warp, then over the warps in order:
    // block_sum_all's order) go to partial[block][ncols]
    auto flush_cols = [&](const double (&acc)[M], const double *nrm) {
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int j = lane + 32 * m;
            if (j < ncols) red[wid * ncols + j] = acc[m];
        }
        if (nrm) {
            const double v = warp_sum(*nrm);
            if (lane == 0) red[NW * ncols + wid] = v;
        }
        __syncthreads();
        for (int j = tid; j < ncols + (nrm ? 1 : 0); j += kSThr) {
            double s = 0.0;
            if (j < ncols)
                for (int w = 0; w < NW; w++) s += red[w * ncols + j];
            else
                for (int w = 0; w < NW; w++) s += red[NW * ncols + w];
            a.partial[(int64_t)bid * a.PS + j] = s;
        }
        __syncthreads();
    };
    auto load_h = [&](const double *h, double (&hreg)[M]) {
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int j = lane + 32 * m;
            hreg[m] = j < ncols ? __ldcg(h + j) : 0.0;
        }
    };
    // PEER: one-shot all-reduce of this rank's CTA partials [.][0, nc) across
    // the ranks (PeerArgs, internal.h).  The warp that owns column j forms the
    // rank's sum in sreduce_cols' order, lane q stores it into slot [par][rank]
    // of rank q's mailbox; every CTA then releases one arrival to every rank
    // and waits for the P x nb arrivals of this reduction on its own counter.
    // Returns this rank's [P][PS] slots of the reduction (summed by the caller).
    unsigned int seq0 = 0, npeer = 0;
    if constexpr (PEER) seq0 = *(volatile const unsigned int *)a.peer->seq;
    auto peer_exchange = [&](int nc) -> const double * {
        const PeerArgs *pa = a.peer;
        const int P = pa->P, PS = pa->PS;
        const unsigned int rs = seq0 + (++npeer);
        const int par = (int)(rs & 1u);
        const int64_t slot = ((int64_t)par * P + pa->rank) * PS;
        for (int j = bid * NW + wid; j < nc; j += nb * NW) {
            double s = 0.0;
            for (int t = lane; t < nb; t += 32) s += __ldcg(a.partial + (int64_t)t * a.PS + j);
            s = warp_sum(s);
            if (lane < P) __stcg(pa->mbox_peer[lane] + slot + j, s);
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence_system();
            for (int q = 0; q < P; q++) red_release_sys_add(pa->ctr_peer[q] + par, 1u);
            const unsigned int target = ((rs + 1u) >> 1) * pa->expect;
            const long long t0 = clock64();
            while (ld_acquire_sys(pa->ctr + par) < target) {
                if (clock64() - t0 > kPeerTimeoutCycles) {
                    a.ctrl->abort_check = a.check;
                    a.ctrl->abort_kind = 2;
                    __threadfence();
                    a.ctrl->abort = 1;
                    break;
                }
            }
            __threadfence();
        }
        __syncthreads();
        return pa->mbox + (int64_t)par * P * PS;
    };
    // sum over the ranks in rank order of entry j of the slots
    auto peer_entry = [&](const double *sl, int j) -> double {
        const PeerArgs *pa = a.peer;
        double s = __ldcg(sl + j);
        for (int q = 1; q < pa->P; q++) s += __ldcg(sl + (int64_t)q * pa->PS + j);
        return s;
    };
    auto peer_h = [&](const double *sl, double (&hreg)[M]) {
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int j = lane + 32 * m;
            hreg[m] = j < ncols ? peer_entry(sl, j) : 0.0;
        }
    };

    const int ph = a.phase;
    double hreg[M];
    // the previous call on this side left its column (the last of this basis)
    // pending: it is formed in this call's first sweep, (w' - Q h2) / beta
    int pend = 0;
    double prb = 0.0;
    {  // (single GPU and multi-GPU peer kernels alike)
        if (a.dst && ncols > 0 && *(volatile const int *)&a.dst->flag) {
            pend = 1;
            prb = a.dst->rbeta;
            if (a.dst->col != ncols - 1) {  // host bookkeeping broken: fail loudly
                if (bid == 0 && tid == 0) {
                    a.ctrl->abort_check = a.check;
                    a.ctrl->abort_kind = 3;
                    __threadfence();
                    a.ctrl->abort = 1;
                }
                return;
            }
        }
    }
    if (a.pre_h && ph <= 1) {  // w -= Q pre_h (restart, Eq. (7))
        load_h(a.pre_h, hreg);
        run_tiles([&](int k, const double *T, const double *W) {
            double s[RPW];
            rowdots(T, hreg, s);
#pragma unroll
            for (int q = 0; q < RPW; q++) {
                const int rr = RPW * wid + q;
                const int64_t r = rb + (int64_t)k * RT + rr;
                if (lane == q * kHalf && r < re) a.w[r] = W[rr] - s[q];
            }
        });
        grid_sync_n(a.flags, a.epoch + (++nbar), nb);
    }

    double nrm_wp = 0.0;
    if (ncols > 0 && ph <= 2) {
        double acc[M];
        if (ph <= 1) {
        // phase A: partial h1
#pragma unroll
        for (int m = 0; m < M; m++) acc[m] = 0.0;
        if (pend) {
            // the pending column pc = ncols - 1: its rows of this tile are formed
            // from the tile itself (row dots with the stored h2 over columns
            // < pc), written back to the basis and used for h1 in place of w'
            const int pc = ncols - 1;
#pragma unroll
            for (int m = 0; m < M; m++) {
                const int j = lane + 32 * m;
                hreg[m] = j < pc ? __ldcg(a.dst->h + j) : 0.0;
            }
            if constexpr (RPW * M > 20 || M > 16) {  // wide bases: the tile is read twice from shared memory
                run_tiles([&](int k, const double *T, const double *W) {
                    double s[RPW];
                    rowdots(T, hreg, s);
                    allrows(s);
#pragma unroll
                    for (int q = 0; q < RPW; q++) {
                        const int rr = RPW * wid + q;
                        const int64_t r = rb + (int64_t)k * RT + rr;
                        const double u = (T[pc * RT + (((rr >> 1) ^ (pc & (kCh - 1))) << 1) + (rr & 1)] - s[q]) * prb;
                        if (lane == q * kHalf && r < re) a.qw[r + (int64_t)pc * a.ldq] = u;
                        const double x = W[rr];
#pragma unroll
                        for (int m = 0; m < M; m++) {
                            const int j = lane + 32 * m;
                            if (colok(m)) acc[m] = fma(j == pc ? u : tval(T, rr, m), x, acc[m]);
                        }
                    }
                });
            } else {  // the tile values read once, kept in registers (as in phase B)
                run_tiles([&](int k, const double *T, const double *W) {
                    double tv[RPW][M], part[RPW];
                    load_tile_rows(T, hreg, tv, part);
                    reduce_rows(part);
                    allrows(part);
#pragma unroll
                    for (int q = 0; q < RPW; q++) {
                        const int rr = RPW * wid + q;
                        const int64_t r = rb + (int64_t)k * RT + rr;
                        const double u = (T[pc * RT + (((rr >> 1) ^ (pc & (kCh - 1))) << 1) + (rr & 1)] - part[q]) * prb;
                        if (lane == q * kHalf && r < re) a.qw[r + (int64_t)pc * a.ldq] = u;
                        const double x = W[rr];
#pragma unroll
                        for (int m = 0; m < M; m++) acc[m] = fma(lane + 32 * m == pc ? u : tv[q][m], x, acc[m]);
                    }
                });
            }
        } else {
        run_tiles([&](int, const double *T, const double *W) {
            if constexpr (RPW == 2) {
                const double x0 = W[2 * wid], x1 = W[2 * wid + 1];
#pragma unroll
                for (int m = 0; m < M; m++)
                    if (colok(m)) {
                        const double2 t = tpair(T, m);
                        acc[m] = fma(t.y, x1, fma(t.x, x0, acc[m]));
                    }
            } else {
#pragma unroll
                for (int q = 0; q < RPW; q++) {
                    const int rr = RPW * wid + q;
                    const double x = W[rr];
#pragma unroll
                    for (int m = 0; m < M; m++)
                        if (colok(m)) acc[m] = fma(tval(T, rr, m), x, acc[m]);
                }
            }
        });
        }
        flush_cols(acc, nullptr);
        if (pend) {  // the formed column rows precede phase B's re-reads of the tiles
            __threadfence();
            __syncthreads();
        }
        if (ph == 0) {
            prefetch();  // phase B re-reads the same tiles: start them under the reduction
            prefetched = true;
        }
        grid_sync_n(a.flags, a.epoch + (++nbar), nb);
        if constexpr (PEER) {
            peer_h(peer_exchange(ncols), hreg);
        } else {
            sreduce_cols(a, ncols, a.h1, bid, nb);
            if (ph == 1) return;  // the host all-reduces h1 across the ranks
            grid_sync_n(a.flags, a.epoch + (++nbar), nb);
            load_h(a.h1, hreg);
        }
        } else {
            load_h(a.h1, hreg);
        }
        // phase B: w' = w - Q h1 (written back), partial h2, ||w'||^2
#pragma unroll
        for (int m = 0; m < M; m++) acc[m] = 0.0;
        if constexpr (RPW * M > 20 || M > 16) {  // wide bases: registers hold acc + hreg only
            run_tiles([&](int k, const double *T, const double *W) {
                double part[RPW];
                rowdots(T, hreg, part);
                allrows(part);
#pragma unroll
                for (int q = 0; q < RPW; q++) {
                    const int rr = RPW * wid + q;
                    const int64_t r = rb + (int64_t)k * RT + rr;
                    const double v = (r < re) ? W[rr] - part[q] : 0.0;
                    if (lane == q * kHalf && r < re) {
                        a.w[r] = v;
                        nrm_wp = fma(v, v, nrm_wp);
                    }
#pragma unroll
                    for (int m = 0; m < M; m++)
                        if (colok(m)) acc[m] = fma(tval(T, rr, m), v, acc[m]);
                }
            });
        } else {  // the tile values read from shared memory once, kept in registers
            run_tiles([&](int k, const double *T, const double *W) {
                double tv[RPW][M], part[RPW];
                load_tile_rows(T, hreg, tv, part);
                reduce_rows(part);
                allrows(part);
#pragma unroll
                for (int q = 0; q < RPW; q++) {
                    const int rr = RPW * wid + q;
                    const int64_t r = rb + (int64_t)k * RT + rr;
                    const double v = (r < re) ? W[rr] - part[q] : 0.0;
                    if (lane == q * kHalf && r < re) {
                        a.w[r] = v;
                        nrm_wp = fma(v, v, nrm_wp);
                    }
#pragma unroll
                    for (int m = 0; m < M; m++) acc[m] = fma(tv[q][m], v, acc[m]);
                }
            });
        }
        flush_cols(acc, &nrm_wp);  // [partial h2, ||w'_b||^2]
    } else if (ph == 0 || ph == 2) {
        run_tiles([&](int k, const double *, const double *W) {
#pragma unroll
            for (int q = 0; q < RPW; q++) {
                const int rr = RPW * wid + q;
                const int64_t r = rb + (int64_t)k * RT + rr;
                if (lane == q * kHalf && r < re) nrm_wp = fma(W[rr], W[rr], nrm_wp);
            }
        });
    }
    const double *sl2 = nullptr;  // PEER: the slots of the [h2; ||w'||^2] exchange
    if (ph == 0 || ph == 2) {
        if (ncols == 0) {
            const double bn = block_sum_all(nrm_wp, sh);
            if (tid == 0) a.partial[(int64_t)bid * a.PS + ncols] = bn;
        }
        if (ncols > 0 && ph == 0 && !a.defer) {  // phase C reads w' written above by this CTA
            __threadfence();
            __syncthreads();
            prefetch();
            prefetched = true;
        }
        grid_sync_n(a.flags, a.epoch + (++nbar), nb);
        if constexpr (PEER) {
            sl2 = peer_exchange(ncols + 1);
        } else {
            sreduce_cols(a, ncols + 1, a.h2, bid, nb);
            if (ph == 2) return;  // the host all-reduces [h2; ||w'||^2] across the ranks
            grid_sync_n(a.flags, a.epoch + (++nbar), nb);
        }
    }
    double nrmp;
    if constexpr (PEER) {
        peer_h(sl2, hreg);
        nrmp = peer_entry(sl2, ncols);
    } else {
        load_h(a.h2, hreg);
        nrmp = __ldcg(a.h2 + ncols);
    }
    // ||h2||^2 from the coefficients every warp already holds (lane: columns
    // lane + 32 m, zeros past ncols); lane 0's butterfly result broadcast, so
    // every thread of every CTA uses the same value
    double hh = 0.0;
#pragma unroll
    for (int m = 0; m < M; m++) hh = fma(hreg[m], hreg[m], hh);
    hh = __shfl_sync(0xffffffffu, warp_sum(hh), 0);
    double beta2 = nrmp - hh;
    const bool pyth = beta2 > 0.5 * nrmp;
    const double amax = a.ctrl->amax[a.check & 1];
    const double thr = 1e-14 * fmax(amax, 1.0);
    bool bd = false;
    double beta = 0.0;
    bool deferred = false;
    if (pyth) {
        beta = sqrt(beta2);
        bd = !(beta > thr);
        if (a.defer && !bd && ncols > 0) {
            // deferred second update: the column keeps w'; the next product reads
            // xs = w' / beta (differs from the final vector by -Q h2 / beta, in
            // span(Q): DESIGN.md 7), the next call on this side forms the column
            const double rbeta = 1.0 / beta;
            for (int64_t r = rb + tid; r < re; r += kSThr) a.xs[r] = __ldcg(a.w + r) * rbeta;
            deferred = true;
        } else if (!bd && ncols > 0) {
            // one reciprocal per kernel instead of a division per row (the
            // division sequence would double this sweep's instruction count)
            const double rbeta = 1.0 / beta;
            run_tiles([&](int k, const double *T, const double *W) {
                double s[RPW];
                rowdots(T, hreg, s);
#pragma unroll
                for (int q = 0; q < RPW; q++) {
                    const int rr = RPW * wid + q;
                    const int64_t r = rb + (int64_t)k * RT + rr;
                    if (lane == q * kHalf && r < re) a.w[r] = (W[rr] - s[q]) * rbeta;
                }
            });
        } else if (!bd) {
            for (int64_t r = rb + tid; r < re; r += kSThr) a.w[r] = a.w[r] / beta;
        }
    } else if (ph == 3) {
        // multi-GPU: the explicit norm of w'' needs one more cross-rank reduction;
        // form w'' and hand the norm to the host (pass-end repair, svdsc.cu)
        if (ncols > 0)
            run_tiles([&](int k, const double *T, const double *W) {
                double s[RPW];
                rowdots(T, hreg, s);
#pragma unroll
                for (int q = 0; q < RPW; q++) {
                    const int rr = RPW * wid + q;
                    const int64_t r = rb + (int64_t)k * RT + rr;
                    if (lane == q * kHalf && r < re) a.w[r] = W[rr] - s[q];
                }
            });
        if (bid == 0 && tid == 0) {
            a.ctrl->abort_check = a.check;
            a.ctrl->abort_kind = 1;
            __threadfence();
            a.ctrl->abort = 1;
        }
        cp_wait<0>();
        return;
    } else {
        double nrm2 = 0.0;
        if (ncols > 0) {
            run_tiles([&](int k, const double *T, const double *W) {
                double s[RPW];
                rowdots(T, hreg, s);
#pragma unroll
                for (int q = 0; q < RPW; q++) {
                    const int rr = RPW * wid + q;
                    const int64_t r = rb + (int64_t)k * RT + rr;
                    if (lane == q * kHalf && r < re) {
                        const double v = W[rr] - s[q];
                        a.w[r] = v;
                        nrm2 = fma(v, v, nrm2);
                    }
                }
            });
        } else {
            for (int64_t r = rb + tid; r < re; r += kSThr) nrm2 = fma(a.w[r], a.w[r], nrm2);
        }
        const double bn = block_sum_all(nrm2, sh);
        if (tid == 0) a.partial[(int64_t)bid * a.PS] = bn;
        grid_sync_n(a.flags, a.epoch + (++nbar), nb);
        if constexpr (PEER) {
            beta = sqrt(fmax(peer_entry(peer_exchange(1), 0), 0.0));
        } else {
            sreduce_cols(a, 1, a.h3, bid, nb);
            grid_sync_n(a.flags, a.epoch + (++nbar), nb);
            beta = sqrt(fmax(__ldcg(a.h3), 0.0));
        }
        bd = !(beta > thr);
        if (!bd)
            for (int64_t r = rb + tid; r < re; r += kSThr) a.w[r] = a.w[r] / beta;
    }
    cp_wait<0>();  // a prefetch may be pending if phase C was skipped
    {
        if (a.dst) {
            if (a.defer && !deferred && !bd) {
                // the final vector was formed here after all (explicit norm, reading
                // G3, or no basis): the next product reads it from xs as planned
                __syncthreads();
                for (int64_t r = rb + tid; r < re; r += kSThr) a.xs[r] = __ldcg(a.w + r);
            }
            if (bid == 0) {
                if (deferred) {
#pragma unroll
                    for (int m = 0; m < M; m++) {
                        const int j = lane + 32 * m;
                        if (wid == 0 && j < ncols) a.dst->h[j] = hreg[m];
                    }
                    if (tid == 0) {
                        a.dst->rbeta = 1.0 / beta;
                        a.dst->col = ncols;
                    }
                }
                if (tid == 0) a.dst->flag = deferred ? 1 : 0;
            }
        }
    }
    if (bid == 0 && tid == 0) {
        // every CTA read seq0 before the first grid barrier, so the next launch
        // is the first to see the advanced count
        if constexpr (PEER) *a.peer->seq = seq0 + npeer;
        if (bd) {
            *a.t_entry = 0.0;
            a.ctrl->amax[(a.check + 1) & 1] = amax;
            a.ctrl->abort_check = a.check;
            __threadfence();
            a.ctrl->abort = 1;
        } else {
            *a.t_entry = beta;
            a.ctrl->amax[(a.check + 1) & 1] = fmax(amax, beta);
        }
    }
}

template <int RT, int NS, int M>
__global__ void __launch_bounds__(512) k_cgs2_stream2(SArgs a) {
    cgs2_stream2_body<RT, NS, M, false>(a, blockIdx.x, gridDim.x);
}
// multi-GPU (peer mailboxes).  grp == NULL: this rank's CTAs are the grid
// (production, one launch per rank); else an emulated multi-rank launch on one
// GPU: CTA group g = blockIdx.x / nb runs rank g with grp[g]
template <int RT, int NS, int M>
__global__ void __launch_bounds__(512) k_cgs2_stream2p(SArgs a) {
    cgs2_stream2_body<RT, NS, M, true>(a, blockIdx.x, gridDim.x);
}
// test support: P ranks emulated as P CTA groups of one cooperative launch
template <int RT, int NS, int M>
__global__ void __launch_bounds__(512) k_cgs2_stream2e(const SArgs *__restrict__ grp, int nb) {
    const int g = blockIdx.x / nb;
    cgs2_stream2_body<RT, NS, M, true>(grp[g], blockIdx.x - g * nb, nb);
}

template <int RT, int NS, int M>
bool launch_stream2(const SArgs &a0, int nsm, cudaStream_t s) {
    SArgs a = a0;
    const size_t smem = ((size_t)NS * stream2_tcols<RT, M>(a.ncols) * RT + NS * RT) * sizeof(double);
    if (smem > 220 * 1024 || a.ncols > 32 * M) return false;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cgs2_stream2<RT, NS, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cgs2_stream2<RT, NS, M>, 512, smem);
    if (bps < 1) return false;
    const int nb = nsm;
    int64_t rpb = (a.N + nb - 1) / nb;
    rpb = (rpb + RT - 1) / RT * RT;
    a.rpb = rpb;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nb, (a.N + rpb - 1) / rpb));
    void *args[] = {&a};
    if (cudaLaunchCooperativeKernel((void *)k_cgs2_stream2<RT, NS, M>, grid, 512, args, smem, s) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    count_launch();
    return true;
}

// ring depth: as many 32-row stages as fit in shared memory up to 192 columns,
// but 4 (not 5) up to 128: with the deferred update's first sweep the 5-stage
// instance spills (80 B) and measured 1-2 % slower (config 3: 982 vs 959 ms);
// 16-row tiles with 4 stages and the register-lean w' sweep were slower, 11a
bool launch_stream2_any(const SArgs &a, int nsm, cudaStream_t s) {
    const int nc = a.ncols;
    if (nc <= 64) return launch_stream2<32, 4, 2>(a, nsm, s);
    if (nc <= 128) return launch_stream2<32, 4, 4>(a, nsm, s);
    if (nc <= 192) return launch_stream2<32, 4, 6>(a, nsm, s);
    if (nc <= 256) return launch_stream2<32, 3, 8>(a, nsm, s);
    if (nc <= 320) return launch_stream2<32, 2, 10>(a, nsm, s);
    if (nc <= 384) return launch_stream2<32, 2, 12>(a, nsm, s);
    if (nc <= 512) return launch_stream2<16, 2, 16>(a, nsm, s);
    if (nc <= 768) return launch_stream2<16, 2, 24>(a, nsm, s);
    return launch_stream2<16, 2, 32>(a, nsm, s);
}

// peer-mailbox streaming CGS2: ngroups = 1 (one rank per GPU, production) or P
// (emulated ranks, grp_dev: device room for P SArgs).  nb CTAs per rank
// whatever its row count (CTAs past the rows contribute zero partials), so
// every rank releases the same number of arrivals (PeerArgs::expect).
template <int RT, int NS, int M>
bool launch_stream2p(SArgs *ga, int ngroups, int nb, void *grp_dev, cudaStream_t s) {
    const int ncols = ga[0].ncols;
    const size_t smem = ((size_t)NS * stream2_tcols<RT, M>(ncols) * RT + NS * RT) * sizeof(double);
    if (smem > 220 * 1024 || ncols > 32 * M || nb < 1) return false;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cgs2_stream2p<RT, NS, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        if constexpr (RT == 32)
            cudaFuncSetAttribute(k_cgs2_stream2e<RT, NS, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    for (int g = 0; g < ngroups; g++) {
        int64_t rpb = (ga[g].N + nb - 1) / nb;
        rpb = std::max<int64_t>(RT, (rpb + RT - 1) / RT * RT);
        ga[g].rpb = rpb;
    }
    cudaError_t e;
    if (!grp_dev) {
        void *args[] = {&ga[0]};
        e = cudaLaunchCooperativeKernel((void *)k_cgs2_stream2p<RT, NS, M>, nb, 512, args, smem, s);
    } else if constexpr (RT == 32) {  // emulation: bases up to 384 columns
        if (cudaMemcpyAsync(grp_dev, ga, ngroups * sizeof(SArgs), cudaMemcpyHostToDevice, s) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        const SArgs *grp = static_cast<const SArgs *>(grp_dev);
        int nbk = nb;
        void *args[] = {&grp, &nbk};
        e = cudaLaunchCooperativeKernel((void *)k_cgs2_stream2e<RT, NS, M>, nb * ngroups, 512, args, smem, s);
    } else {
        return false;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    count_launch();
    return true;
}
bool launch_stream2p_any(SArgs *ga, int ngroups, int nb, void *grp_dev, cudaStream_t s) {
    const int nc = ga[0].ncols;
    if (nc <= 64) return launch_stream2p<32, 4, 2>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 128) return launch_stream2p<32, 5, 4>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 192) return launch_stream2p<32, 4, 6>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 256) return launch_stream2p<32, 3, 8>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 320) return launch_stream2p<32, 2, 10>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 384) return launch_stream2p<32, 2, 12>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 512) return launch_stream2p<16, 2, 16>(ga, ngroups, nb, grp_dev, s);
    if (nc <= 768) return launch_stream2p<16, 2, 24>(ga, ngroups, nb, grp_dev, s);
    return launch_stream2p<16, 2, 32>(ga, ngroups, nb, grp_dev, s);
}

// ---------------------------------------------------------------------------
// TMA variant (B200-native), warp-specialized producer/consumer pipeline.
//   * A row tile is 32 rows x ncols: ceil(ncols/16) TMA boxes of 32 rows x 16
//     columns (column-major, no swizzle: a column segment is 256 contiguous
//     bytes; 16-row segments measured ~10% less HBM bandwidth, tools/tma_bw.cu)
//     plus one 256-byte bulk copy of the tile's w rows, completing on the
//     stage's `full` mbarrier.  One producer thread issues the copies; the 16
//     consumer warps release a stage by arriving on its `empty` mbarrier, so the
//     producer runs up to ns stages ahead and consumers never wait for each
//     other to free a buffer.
//   * Consumer warp w owns columns [w M, w M + M); lane = row of the tile.
//     Column dots (Q^T w) accumulate per thread over the CTA's rows and are
//     reduced over the 32 lanes once per sweep.  Row dots (Q h) are per-thread
//     partials over the warp's columns, combined over the 16 warps through a
//     double-buffered shared array and ONE named barrier per tile; every warp
//     then sums the 16 partials of its rows itself (no shuffles per row).
//   * Phase B keeps the thread's Q values in registers between the row dot
//     (w' = w - Q h1) and the column dot (Q^T w'): Q is read from shared
//     memory once per sweep.
//   * Sweeps alternate direction so that each sweep starts on the tiles the
//     previous one read last (still in L2).
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// named barrier over the 16 warps (row-dot partial exchange)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

constexpr int kTmaNW = 16;           // warps; thread 0 also issues the copies
constexpr int kTmaThreads = kTmaNW * 32;  // 4 warps per SMSP: up to 128 registers per thread
                                           // (a 17th, producer-only warp capped them at 96)
constexpr int kTmaRT = 32;           // rows per tile
constexpr int kTmaMaxNS = 8;

template <int M>
__global__ void __launch_bounds__(kTmaThreads, 1) k_cgs2_tma(const __grid_constant__ CUtensorMap tq, SArgs a, int ns,
                                                             int nsplit) {
    constexpr int RT = kTmaRT, NW = kTmaNW, J = M;
    grid_prepare(a.flags, a.epoch);
    if (*(volatile int *)&a.ctrl->abort) return;
    if (a.gate && *(volatile const int *)a.gate != a.gate_want) return;  // PRO gate, uniform
    unsigned int nbar = 0;
    extern __shared__ __align__(128) double smem_raw[];
    __shared__ __align__(8) uint64_t full[kTmaMaxNS], empty[kTmaMaxNS];
    __shared__ double sh[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr bool producer = false;  // no producer-only warp
    const int ptid = 0;               // the thread that issues the copies
    const int ncols = a.ncols;
    const int nbox = (ncols + 15) >> 4;
    // a tile is split into nsplit column groups, each its own pipeline unit
    // (stage): warps [g NW/nsplit, (g+1) NW/nsplit) own the group's columns,
    // so more, smaller units are in flight per tile (a full-width 32 x 300
    // tile is 77 KB: only two fit)
    const int wpg = NW / nsplit;            // warps per group
    const int gbox = wpg * M / 16;          // boxes per group
    const int grp = wid / wpg;              // this warp's group
    const int stage_d = gbox * 512 + RT;    // doubles per unit: boxes, then the tile's w rows
    double *smem_t = smem_raw;
    double *rpart = smem_t + (size_t)ns * stage_d;  // [2][NW][RT] row-dot partials
    double *hs = rpart + 2 * NW * RT;               // coefficient vector of the current sweep (ncols)
    const int64_t rb = (int64_t)blockIdx.x * a.rpb;
    const int64_t re = min(a.N, rb + a.rpb);
    const int ntiles = rb < re ? (int)((re - rb + RT - 1) / RT) : 0;
    const int nunits = ntiles * nsplit;
    if (tid == ptid) {
        for (int q = 0; q < ns; q++) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], wpg);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // producer state (meaningful in the producer thread only)
    int g_issue = 0, u_issued = 0;
    int sweep_no = 0;
    auto tile_of = [&](int k) { return (sweep_no & 1) ? ntiles - 1 - k : k; };
    auto issue_next = [&]() {  // producer thread: next unit of the current sweep into the ring
        const int st = g_issue % ns;
        if (g_issue >= ns) mbar_wait(&empty[st], (unsigned)(((g_issue / ns) - 1) & 1));
        const int k = u_issued / nsplit, g = u_issued % nsplit;
        const int64_t r0 = rb + (int64_t)tile_of(k) * RT;
        const int b0 = g * gbox, b1 = min(nbox, b0 + gbox);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[st], (unsigned)(max(0, b1 - b0) * 4096 + RT * 8));
        double *dst = smem_t + (size_t)st * stage_d;
        for (int b = b0; b < b1; b++) tma_load_2d(dst + (b - b0) * 512, &tq, (int)r0, 16 * b, &full[st]);
        bulk_load(dst + gbox * 512, a.w + r0, RT * 8, &full[st]);
        g_issue++;
        u_issued++;
    };
    auto prefetch = [&]() {  // first units of the current sweep (before a grid barrier)
        if (tid == ptid)
            while (u_issued < nunits && u_issued < ns) issue_next();
    };
    // consumer: unit of tile k for this warp's group is global use index
    // base + k nsplit + grp (units are issued in that order)
    int use_base = 0;
    auto run_tiles = [&](auto &&body) {
        if (ntiles > 0) {
            for (int k = 0; k < ntiles; k++) {
                // keep ns units in flight: unit u goes into the stage of unit
                // u - ns (a tile <= k - 1), released before tile k is entered
                if (tid == ptid)
                    while (u_issued < nunits && u_issued < k * nsplit + ns) issue_next();
                const int gu = use_base + k * nsplit + grp;
                const int st = gu % ns;
                mbar_wait(&full[st], (unsigned)((gu / ns) & 1));
                const double *T = smem_t + (size_t)st * stage_d;
                body(tile_of(k), k, T, T + gbox * 512);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
            }
        }
        use_base += nunits;
        sweep_no++;
        u_issued = 0;
    };
    // element of the thread's row (lane) and column w M + j
    const int row = lane;
    auto colof = [&](int j) { return wid * M + j; };
    auto qaddr = [&](int j) {  // within the group's stage
        const int c = colof(j) - grp * wpg * M;
        return ((c >> 4) << 9) + ((c & 15) << 5) + row;
    };
    auto load_q = [&](const double *T, double (&q)[J]) {
#pragma unroll
        for (int j = 0; j < J; j++) q[j] = colof(j) < ncols ? T[qaddr(j)] : 0.0;
    };
    // coefficients to shared memory (every thread of the CTA takes part: call
    // between CTA-wide barriers); read back as warp-broadcast loads
    auto load_h = [&](const double *h) {
        for (int j = tid; j < ncols; j += kTmaThreads) hs[j] = __ldcg(h + j);
        __syncthreads();
    };
    // row dot over all columns for the tile row of this lane (valid in every
    // consumer thread after one named barrier)
    auto row_dot = [&](int k, const double (&q)[J]) -> double {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int j = 0; j < J; j += 2) {
            if (colof(j) < ncols) s0 = fma(q[j], hs[colof(j)], s0);
            if (j + 1 < J && colof(j + 1) < ncols) s1 = fma(q[j + 1], hs[colof(j + 1)], s1);
        }
        const double s = s0 + s1;
        double *rp = rpart + (k & 1) * NW * RT;
        rp[wid * RT + row] = s;
        consumers_sync();
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < NW; w++) t += rp[w * RT + row];
        return t;
    };
    // column sums of the per-thread accumulators -> partial[block][c]
    auto flush_cols = [&](double (&acc)[J]) {
        if (!producer) {
#pragma unroll
            for (int j = 0; j < J; j++) {
                double v = acc[j];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0 && colof(j) < ncols) a.partial[(int64_t)blockIdx.x * a.PS + colof(j)] = v;
            }
        }
    };

    if (a.pre_h) {  // w -= Q pre_h (restart, Eq. (7))
        load_h(a.pre_h);
        run_tiles([&](int kt, int k, const double *T, const double *W) {
            double q[J];
            load_q(T, q);
            const double s = row_dot(k, q);
            const int64_t r = rb + (int64_t)kt * RT + row;
            if (wid == NW - 1 && r < re) a.w[r] = W[row] - s;
        });
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        grid_sync(a.flags, a.epoch + (++nbar));
    }

    double nrm_wp = 0.0;
    if (ncols > 0) {
        double acc[J];
#pragma unroll
        for (int j = 0; j < J; j++) acc[j] = 0.0;
        // phase A: partial h1 = Q_b^T w_b
        run_tiles([&](int kt, int, const double *T, const double *W) {
            const int64_t r = rb + (int64_t)kt * RT + row;
            const double x = r < re ? W[row] : 0.0;
#pragma unroll
            for (int j = 0; j < J; j++)
                if (colof(j) < ncols) acc[j] = fma(T[qaddr(j)], x, acc[j]);
        });
        flush_cols(acc);
        prefetch();
        grid_sync(a.flags, a.epoch + (++nbar));
        sreduce_cols(a, ncols, a.h1, blockIdx.x, gridDim.x);
        grid_sync(a.flags, a.epoch + (++nbar));
        load_h(a.h1);
#pragma unroll
        for (int j = 0; j < J; j++) acc[j] = 0.0;
        // phase B: w' = w - Q h1 (written back), partial h2 = Q^T w', ||w'||^2
        run_tiles([&](int kt, int k, const double *T, const double *W) {
            double q[J];
            load_q(T, q);
            const double s = row_dot(k, q);
            const int64_t r = rb + (int64_t)kt * RT + row;
            const double v = (r < re) ? W[row] - s : 0.0;
            if (wid == NW - 1 && r < re) {
                a.w[r] = v;
                nrm_wp = fma(v, v, nrm_wp);
            }
#pragma unroll
            for (int j = 0; j < J; j++) acc[j] = fma(q[j], v, acc[j]);
        });
        flush_cols(acc);
    } else {
        run_tiles([&](int kt, int, const double *, const double *W) {
            const int64_t r = rb + (int64_t)kt * RT + row;
            if (wid == NW - 1 && r < re) nrm_wp = fma(W[row], W[row], nrm_wp);
        });
    }
    {
        const double bn = block_sum_all(nrm_wp, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS + ncols] = bn;
    }
    if (ncols > 0) {  // phase C reads w' written above by this CTA (generic -> async proxy)
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncthreads();
        prefetch();
    }
    grid_sync(a.flags, a.epoch + (++nbar));
    sreduce_cols(a, ncols + 1, a.h2, blockIdx.x, gridDim.x);
    grid_sync(a.flags, a.epoch + (++nbar));
    load_h(a.h2);
    const double nrmp = __ldcg(a.h2 + ncols);
    double hh = 0.0;
    for (int j = tid; j < ncols; j += kTmaThreads) hh = fma(hs[j], hs[j], hh);
    hh = block_sum_all(hh, sh);
    double beta2 = nrmp - hh;
    const bool pyth = beta2 > 0.5 * nrmp;
    const double amax = a.ctrl->amax[a.check & 1];
    const double thr = 1e-14 * fmax(amax, 1.0);
    bool bd = false;
    double beta = 0.0;
    if (pyth) {
        beta = sqrt(beta2);
        bd = !(beta > thr);
        if (!bd && ncols > 0) {
            run_tiles([&](int kt, int k, const double *T, const double *W) {
                double q[J];
                load_q(T, q);
                const double s = row_dot(k, q);
                const int64_t r = rb + (int64_t)kt * RT + row;
                if (wid == NW - 1 && r < re) a.w[r] = (W[row] - s) / beta;
            });
        } else if (!bd) {
            for (int64_t r = rb + tid; r < re; r += kTmaThreads) a.w[r] = a.w[r] / beta;
        }
    } else {
        double nrm2 = 0.0;
        if (ncols > 0) {
            run_tiles([&](int kt, int k, const double *T, const double *W) {
                double q[J];
                load_q(T, q);
                const double s = row_dot(k, q);
                const int64_t r = rb + (int64_t)kt * RT + row;
                if (wid == NW - 1 && r < re) {
                    const double v = W[row] - s;
                    a.w[r] = v;
                    nrm2 = fma(v, v, nrm2);
                }
            });
        } else {
            for (int64_t r = rb + tid; r < re; r += kTmaThreads) nrm2 = fma(a.w[r], a.w[r], nrm2);
        }
        const double bn = block_sum_all(nrm2, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS] = bn;
        grid_sync(a.flags, a.epoch + (++nbar));
        sreduce_cols(a, 1, a.h3, blockIdx.x, gridDim.x);
        grid_sync(a.flags, a.epoch + (++nbar));
        beta = sqrt(fmax(__ldcg(a.h3), 0.0));
        bd = !(beta > thr);
        if (!bd)
            for (int64_t r = rb + tid; r < re; r += kTmaThreads) a.w[r] = a.w[r] / beta;
    }
    // phase C prefetched but skipped (breakdown): wait for those copies so
    // that no bulk copy is in flight when the CTA exits
    if (tid == ptid && ncols > 0 && pyth && bd) {
        for (int gu = use_base; gu < use_base + min(nunits, ns); gu++)
            mbar_wait(&full[gu % ns], (unsigned)((gu / ns) & 1));
    }
    if (blockIdx.x == 0 && tid == 0) {
        if (bd) {
            *a.t_entry = 0.0;
            a.ctrl->amax[(a.check + 1) & 1] = amax;
            a.ctrl->abort_check = a.check;
            __threadfence();
            a.ctrl->abort = 1;
        } else {
            *a.t_entry = beta;
            a.ctrl->amax[(a.check + 1) & 1] = fmax(amax, beta);
        }
    }
}

template <int M>
bool launch_tma(const CUtensorMap &tq, const SArgs &a0, int nsm, cudaStream_t s) {
    SArgs a = a0;
    if (a.ncols > kTmaNW * M) return false;
    // one column group per tile (splitting tiles into column-group units for a
    // deeper ring measured slower)
    const int nsplit = 1;
    const int gbox = (kTmaNW / nsplit) * M / 16;
    const size_t stage_b = ((size_t)gbox * 512 + kTmaRT) * sizeof(double);
    const size_t fixed = ((size_t)2 * kTmaNW * kTmaRT + a.ncols + 2) * sizeof(double) + 128;
    const int ns = (int)std::min<size_t>(kTmaMaxNS, (200 * 1024 - fixed) / stage_b);
    if (ns < 2 * nsplit) return false;
    const size_t smem = ns * stage_b + fixed;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cgs2_tma<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cgs2_tma<M>, kTmaThreads, smem);
    if (bps < 1) return false;
    const int nb = nsm;
    int64_t rpb = (a.N + nb - 1) / nb;
    rpb = (rpb + kTmaRT - 1) / kTmaRT * kTmaRT;
    a.rpb = rpb;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nb, (a.N + rpb - 1) / rpb));
    CUtensorMap map = tq;
    void *args[] = {&map, &a, (void *)&ns, (void *)&nsplit};
    if (cudaLaunchCooperativeKernel((void *)k_cgs2_tma<M>, grid, kTmaThreads, args, smem, s) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    count_launch();
    return true;
}

bool launch_tma_any(const CUtensorMap &tq, const SArgs &a, int nsm, cudaStream_t s) {
    const int nc = a.ncols;
    if (nc <= 16 * 2) return launch_tma<2>(tq, a, nsm, s);
    if (nc <= 16 * 4) return launch_tma<4>(tq, a, nsm, s);
    if (nc <= 16 * 8) return launch_tma<8>(tq, a, nsm, s);
    if (nc <= 16 * 12) return launch_tma<12>(tq, a, nsm, s);
    if (nc <= 16 * 16) return launch_tma<16>(tq, a, nsm, s);
    if (nc <= 16 * 20) return launch_tma<20>(tq, a, nsm, s);
    if (nc <= 16 * 24) return launch_tma<24>(tq, a, nsm, s);
    return false;  // wider bases: cp.async variants
}

}  // namespace

bool make_basis_tmap(void *map128, const double *base, int64_t N, int64_t ncols_total, int64_t ld) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
    }
    if (!encode || (ld % 2) || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)ncols_total};
    cuuint64_t gstride[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {32, 16};  // 32 rows x 16 columns (k_cgs2_tma row tile)
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap *>(map128), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                        const_cast<double *>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------
// Single-cluster CGS2 for small bases (BASELINE config 1, the V side of config
// 2): C <= 16 CTAs of one thread-block cluster own contiguous row blocks; Q is
// read from L2 (it is L2-resident between calls at these sizes), w lives in
// shared memory, and each global reduction is an all-gather of the C partial
// vectors through distributed shared memory + one cluster barrier (hardware,
// sub-microsecond) instead of two grid barriers and a reduction kernel phase.
// Every CTA sums the C partials in the same fixed order: bitwise identical
// coefficients everywhere, deterministic.
constexpr int kClThreads = 512;
struct CArgs {
    int64_t N;
    int ncols;
    const double *Q;
    int64_t ldq;
    double *w;
    Ctrl *ctrl;
    double *t_entry;
    int check;
    const double *pre_h;
    PreReduce pre;
    int rpb;  // rows per CTA
    unsigned int *flags;  // grid-barrier slots: this launch zeroes the next launch's slot
    unsigned int epoch;
    const int *gate;      // partial re-orthogonalization gate (FusedScratch::gate)
    int gate_want;
    int qstage;           // 1: the CTA's rows of Q are staged in shared memory once (read from L2 once, not 3x)
};

__global__ void __launch_bounds__(kClThreads) k_cgs2_cluster(CArgs a) {
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NWc = kClThreads / 32;
    const int ncols = a.ncols, PS = ncols + 2;
    extern __shared__ __align__(16) double csm[];
    double *ws = csm;                       // rpb: this CTA's rows of w
    double *hs = ws + a.rpb;                // PS: reduced coefficients
    double *part = hs + PS;                 // 3 x PS: partial vectors (one buffer per reduction)
    double *qs = part + 3 * PS;             // qstage: ncols x rpb, column-major (this CTA's rows of Q)
    __shared__ double sh[32];
    const int64_t r0 = (int64_t)me * a.rpb;
    const int nr = (int)max((int64_t)0, min((int64_t)a.rpb, a.N - r0));
    const double *Qb = a.Q + r0;
    const bool staged = a.qstage != 0;
    // Q was written before the stream predecessor (the product) started: it is
    // staged before the PDL wait, under the predecessor's tail
    if (staged) {  // 16-byte copies (rpb and ldq are even: every column segment is aligned)
        const int half = (nr + 1) / 2;
        for (int j = wid; j < ncols; j += NWc)
            for (int c2 = lane; c2 < half; c2 += 32) {
                const int rem = nr - 2 * c2;
                const unsigned sa = (unsigned)__cvta_generic_to_shared(qs + (int64_t)j * a.rpb + 2 * c2);
                const double *src = Qb + (int64_t)j * a.ldq + 2 * c2;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src),
                             "r"(rem >= 2 ? 16 : 8)
                             : "memory");
            }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    pdl_wait();  // launched with launch_pdl: w (and ctrl) are the predecessor's output
    pdl_trigger();
    grid_prepare(a.flags, a.epoch);  // keep the barrier-slot chain of the fused launches intact
    if (*(volatile int *)&a.ctrl->abort || (a.gate && *(volatile const int *)a.gate != a.gate_want)) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;  // uniform over the cluster (abort / PRO gate)
    }
    for (int i = tid; i < nr; i += kClThreads) {
        double x;
        if (a.pre.partial) {  // finish a dense split-K product (k_split_reduce order)
            x = 0.0;
            for (int q = 0; q < a.pre.splits; q++) x += a.pre.partial[q * a.N + r0 + i];
            if (a.pre.yprev) x -= *a.pre.c_dev * a.pre.yprev[r0 + i];
        } else {
            x = a.w[r0 + i];
        }
        ws[i] = x;
    }
    if (staged) asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // Q(i, j) of the CTA's rows: shared memory when staged, else L2
    auto qv = [&](int i, int j) -> double {
        return staged ? qs[(int64_t)j * a.rpb + i] : __ldg(Qb + i + (int64_t)j * a.ldq);
    };
    // column dots of Q_b^T v (v in shared memory) -> part buffer pb[0..ncols)
    auto coldots = [&](const double *v, double *pb) {
        for (int j = wid; j < ncols; j += NWc) {
            double s0 = 0.0, s1 = 0.0;
            int i = lane;
            for (; i + 32 < nr; i += 64) {
                s0 = fma(qv(i, j), v[i], s0);
                s1 = fma(qv(i + 32, j), v[i + 32], s1);
            }
            if (i < nr) s0 = fma(qv(i, j), v[i], s0);
            double t = s0 + s1;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            if (lane == 0) pb[j] = t;
        }
    };
    // v[i] -= sum_j Q[i][j] h[j] for the CTA's rows (thread per row, coalesced over rows)
    auto rowupdate = [&](double *v, const double *h, double *nrm) {
        for (int i = tid; i < nr; i += kClThreads) {
            double s0 = 0.0, s1 = 0.0;
            int j = 0;
            for (; j + 1 < ncols; j += 2) {
                s0 = fma(qv(i, j), h[j], s0);
                s1 = fma(qv(i, j + 1), h[j + 1], s1);
            }
            if (j < ncols) s0 = fma(qv(i, j), h[j], s0);
            const double x = v[i] - (s0 + s1);
            v[i] = x;
            if (nrm) *nrm = fma(x, x, *nrm);
        }
    };
    // all CTAs: hs[0..cnt) = sum over the cluster's partial buffers (fixed order)
    auto allreduce = [&](int buf, int cnt) {
        cl.sync();  // every CTA's partials written
        for (int j = tid; j < cnt; j += kClThreads) {
            double t = 0.0;
            for (int c = 0; c < C; c++) t += cl.map_shared_rank(part + buf * PS, c)[j];
            hs[j] = t;
        }
        __syncthreads();
    };
    auto blocksum = [&](double v) -> double {
        v = warp_sum(v);
        __syncthreads();
        if (lane == 0) sh[wid] = v;
        __syncthreads();
        double t = 0.0;
        for (int q = 0; q < NWc; q++) t += sh[q];
        __syncthreads();
        return t;
    };
    if (a.pre_h) {  // w -= Q pre_h (restart, Eq. (7))
        for (int j = tid; j < ncols; j += kClThreads) hs[j] = a.pre_h[j];
        __syncthreads();
        rowupdate(ws, hs, nullptr);
        __syncthreads();
    }
    double nrm_wp = 0.0;
    if (ncols > 0) {
        coldots(ws, part);  // phase A: partial h1
        allreduce(0, ncols);
        rowupdate(ws, hs, &nrm_wp);  // phase B: w' = w - Q h1
        __syncthreads();
        coldots(ws, part + PS);      // partial h2
    } else {
        for (int i = tid; i < nr; i += kClThreads) nrm_wp = fma(ws[i], ws[i], nrm_wp);
    }
    {
        const double bn = blocksum(nrm_wp);
        if (tid == 0) part[PS + ncols] = bn;
    }
    allreduce(1, ncols + 1);
    const double nrmp = hs[ncols];
    double hh = 0.0;
    for (int j = tid; j < ncols; j += kClThreads) hh = fma(hs[j], hs[j], hh);
    hh = blocksum(hh);
    double beta2 = nrmp - hh;
    const bool pyth = beta2 > 0.5 * nrmp;
    double nrm2 = 0.0;
    if (ncols > 0) rowupdate(ws, hs, pyth ? nullptr : &nrm2);  // phase C: w'' = w' - Q h2
    __syncthreads();
    if (!pyth) {  // explicit norm (uniform branch)
        const double bn = blocksum(nrm2);
        if (tid == 0) part[2 * PS] = bn;
        allreduce(2, 1);
        beta2 = hs[0];
    }
    const double beta = sqrt(fmax(beta2, 0.0));
    const double amax = a.ctrl->amax[a.check & 1];
    const bool bd = !(beta > 1e-14 * fmax(amax, 1.0));
    if (me == 0 && tid == 0) {
        if (bd) {
            *a.t_entry = 0.0;
            a.ctrl->amax[(a.check + 1) & 1] = amax;
            a.ctrl->abort_check = a.check;
            __threadfence();
            a.ctrl->abort = 1;
        } else {
            *a.t_entry = beta;
            a.ctrl->amax[(a.check + 1) & 1] = fmax(amax, beta);
        }
    }
    if (!bd)
        for (int i = tid; i < nr; i += kClThreads) a.w[r0 + i] = ws[i] / beta;
    cl.sync();  // no CTA exits while its shared memory may still be read remotely
}

// ---------------------------------------------------------------------------
// Cluster CGS2 for narrow small bases (ncols <= 32 MC, basis <= 2 MB: BASELINE
// config 1).  Same 16-CTA cluster and row blocks as k_cgs2_cluster, every
// phase arranged for latency (the call is ~20 dependent phases of a few hundred
// cycles each, not a bandwidth problem):
//  * Q staged with 8-byte cp.async into an odd-stride column-major block
//    BEFORE the PDL wait, i.e. under the product's tail;
//  * column dots: warp w owns a slab of rows, lane l columns l + 32 m (odd
//    stride: conflict-free), cross-warp sums through shared memory;
//  * cluster all-reduce by push: the thread that forms entry j of the CTA's
//    partial vector stores it into slot [me] of every CTA's receive buffer
//    (DSMEM stores), one cluster barrier (release / acquire), then every CTA
//    sums the C slots locally in rank order (bitwise identical everywhere, no
//    remote loads after the barrier);
//  * ||w'||^2 rides in the h2 vector; ||h2||^2 is summed by every thread itself.
template <int MC>
__global__ void __launch_bounds__(kClThreads) k_cgs2_cl(CArgs a) {
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = kClThreads / 32;
    const int ncols = a.ncols, PS = ncols + 2, qld = a.rpb | 1;
    extern __shared__ __align__(16) double csm[];
    double *ws = csm;                   // rpb: this CTA's rows of w
    double *hs = ws + a.rpb;            // PS: reduced vector
    double *red = hs + PS;              // NW x PS: per-warp column sums
    double *recv = red + NW * PS;       // 3 x C x PS: pushed CTA partials, one set per reduction
    double *qs = recv + 3 * C * PS;     // ncols x qld: this CTA's rows of Q
    __shared__ double sh[NW];
    __shared__ __align__(8) uint64_t rbar[3];  // one per reduction: completes when all C pushes landed
    const int64_t r0 = (int64_t)me * a.rpb;
    const int nr = (int)max((int64_t)0, min((int64_t)a.rpb, a.N - r0));
    const double *Qb = a.Q + r0;
    // Q was final before the stream predecessor (the product) started
    for (int j = wid; j < ncols; j += NW)
        for (int i = lane; i < nr; i += 32) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(qs + (int64_t)j * qld + i);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(Qb + (int64_t)j * a.ldq + i)
                         : "memory");
        }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // receive barriers armed for the byte counts of the three reductions; the
    // cluster barrier that publishes their initialization is awaited just
    // before the first push
    if (tid == 0) {
        for (int r = 0; r < 3; r++) mbar_init(&rbar[r], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&rbar[0], (unsigned)(C * ncols * 8));
        mbar_expect_tx(&rbar[1], (unsigned)(C * (ncols + 1) * 8));
        mbar_expect_tx(&rbar[2], (unsigned)(C * 8));
    }
    cl.barrier_arrive();
    bool joined = false;
    pdl_wait();  // launched with launch_pdl: w (and ctrl) are the predecessor's output
    pdl_trigger();
    grid_prepare(a.flags, a.epoch);  // keep the barrier-slot chain of the fused launches intact
    if (*(volatile int *)&a.ctrl->abort || (a.gate && *(volatile const int *)a.gate != a.gate_want)) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        cl.barrier_wait();  // (nothing is pushed: uniform over the cluster)
        return;  // abort / PRO gate
    }
    for (int i = tid; i < nr; i += kClThreads) {
        double x;
        if (a.pre.partial) {  // finish a dense split-K product (k_split_reduce order)
            x = 0.0;
            for (int q = 0; q < a.pre.splits; q++) x += a.pre.partial[q * a.N + r0 + i];
            if (a.pre.yprev) x -= *a.pre.c_dev * a.pre.yprev[r0 + i];
        } else {
            x = a.w[r0 + i];
        }
        ws[i] = x;
    }
    if (a.pre_h)
        for (int j = tid; j < ncols; j += kClThreads) hs[j] = a.pre_h[j];
    const double amax = a.ctrl->amax[a.check & 1];  // (loaded early: off the tail's critical path)
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // ws[i] -= sum_j Q(i, j) hs[j] (thread per row: unit stride in qs)
    auto rowupdate = [&](double *nrm) {
        for (int i = tid; i < nr; i += kClThreads) {
            double s0 = 0.0, s1 = 0.0;
            int j = 0;
            for (; j + 1 < ncols; j += 2) {
                s0 = fma(qs[(int64_t)j * qld + i], hs[j], s0);
                s1 = fma(qs[(int64_t)(j + 1) * qld + i], hs[j + 1], s1);
            }
            if (j < ncols) s0 = fma(qs[(int64_t)j * qld + i], hs[j], s0);
            const double x = ws[i] - (s0 + s1);
            ws[i] = x;
            if (nrm) *nrm = fma(x, x, *nrm);
        }
    };
    // push value t into slot [me] entry j of reduction set r of every CTA
    // (st.async: the store completes on the receiver's mbarrier rbar[r])
    // (every thread has joined the initialization barrier before its first push)
    auto push = [&](int r, int j, double t) {
        const unsigned la = smem_u32(recv + (int64_t)(r * C + me) * PS + j), lb = smem_u32(&rbar[r]);
        for (int c = 0; c < C; c++) {
            unsigned ra, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(c));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(c));
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra),
                         "d"(t), "r"(rb)
                         : "memory");
        }
    };
    // CTA partial of Q_b^T ws (+ ||ws_b||^2 in entry ncols when with_norm),
    // pushed into reduction set r of every CTA; once all C pushes landed hs =
    // the cluster sum in rank order
    const int rs = (nr + NW - 1) / NW, i0 = min(nr, wid * rs), i1 = min(nr, i0 + rs);
    auto coldots_allreduce = [&](int r, bool with_norm) {
        double acc[MC];
#pragma unroll
        for (int m = 0; m < MC; m++) acc[m] = 0.0;
        double nrm = 0.0;
#pragma unroll 4
        for (int i = i0; i < i1; i++) {
            const double x = ws[i];
#pragma unroll
            for (int m = 0; m < MC; m++) {
                const int j = lane + 32 * m;
                if (j < ncols) acc[m] = fma(qs[(int64_t)j * qld + i], x, acc[m]);
            }
            nrm = fma(x, x, nrm);
        }
#pragma unroll
        for (int m = 0; m < MC; m++) {
            const int j = lane + 32 * m;
            if (j < ncols) red[wid * PS + j] = acc[m];
        }
        if (with_norm && lane == 0) red[wid * PS + ncols] = nrm;
        __syncthreads();
        const int cnt = ncols + (with_norm ? 1 : 0);
        if (!joined) {
            cl.barrier_wait();
            joined = true;
        }
        for (int j = tid; j < cnt; j += kClThreads) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;  // fixed order: ((w0+w4+..) + (w1+..)) + ...
#pragma unroll
            for (int w = 0; w < NW; w += 4) {
                t0 += red[w * PS + j];
                t1 += red[(w + 1) * PS + j];
                t2 += red[(w + 2) * PS + j];
                t3 += red[(w + 3) * PS + j];
            }
            push(r, j, (t0 + t1) + (t2 + t3));
        }
        mbar_wait(&rbar[r], 0);  // all C pushes landed
        for (int j = tid; j < cnt; j += kClThreads) {
            double t = 0.0;
            for (int c = 0; c < C; c++) t += recv[(int64_t)(r * C + c) * PS + j];
            hs[j] = t;
        }
        __syncthreads();
    };
    if (a.pre_h) {  // w -= Q pre_h (restart, Eq. (7))
        rowupdate(nullptr);
        __syncthreads();
    }
    if (ncols > 0) {
        coldots_allreduce(0, false);  // h1
        rowupdate(nullptr);           // w' = w - Q h1
        __syncthreads();
    }
    coldots_allreduce(1, true);  // [h2; ||w'||^2]
    const double nrmp = hs[ncols];
    double hh = 0.0;
    {  // every thread, same order (four chains)
        double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0;
        int j = 0;
        for (; j + 3 < ncols; j += 4) {
            h0 = fma(hs[j], hs[j], h0);
            h1 = fma(hs[j + 1], hs[j + 1], h1);
            h2 = fma(hs[j + 2], hs[j + 2], h2);
            h3 = fma(hs[j + 3], hs[j + 3], h3);
        }
        for (; j < ncols; j++) h0 = fma(hs[j], hs[j], h0);
        hh = (h0 + h1) + (h2 + h3);
    }
    double beta2 = nrmp - hh;
    const bool pyth = beta2 > 0.5 * nrmp;
    double nrm2 = 0.0;
    if (ncols > 0) rowupdate(pyth ? nullptr : &nrm2);  // w'' = w' - Q h2
    if (!pyth) {  // explicit norm (uniform branch): block sum, then a third push all-reduce
        nrm2 = warp_sum(nrm2);
        if (lane == 0) sh[wid] = nrm2;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int q = 0; q < NW; q++) t += sh[q];
            push(2, 0, t);
        }
        mbar_wait(&rbar[2], 0);
        double t = 0.0;
        for (int c = 0; c < C; c++) t += recv[(int64_t)(2 * C + c) * PS];
        beta2 = t;
    } else {
        __syncthreads();
    }
    const double beta = sqrt(fmax(beta2, 0.0));
    const bool bd = !(beta > 1e-14 * fmax(amax, 1.0));
    if (me == 0 && tid == 0) {
        if (bd) {
            *a.t_entry = 0.0;
            a.ctrl->amax[(a.check + 1) & 1] = amax;
            a.ctrl->abort_check = a.check;
            __threadfence();
            a.ctrl->abort = 1;
        } else {
            *a.t_entry = beta;
            a.ctrl->amax[(a.check + 1) & 1] = fmax(amax, beta);
        }
    }
    if (!bd) {
        const double rbeta = 1.0 / beta;
        for (int i = tid; i < nr; i += kClThreads) a.w[r0 + i] = ws[i] * rbeta;
    }
    // every push into this CTA landed before its last mbarrier wait: CTAs may exit
}

// returns false if the fused path cannot be used (caller falls back)
bool cgs2_fused(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
                const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nsm, cudaStream_t s,
                const void *tmap) {
    // kernel choice (SVDSC_POLICY_CGS2): 0 automatic by size -- one thread-block
    // cluster for bases <= 2 MB, else the Q-resident cooperative kernel when the
    // CTA's rows of Q fit in shared memory, else the cp.async streaming kernel;
    // 2 / 3 / 4 / 5 force Q-resident / streaming / TMA streaming / cluster;
    // 1 (split kernels) and an inapplicable forced kernel return false
    const int pol = g_policy.cgs2;
    if (pol == 1) return false;
    constexpr int kThreads = 256;
    const size_t smem_cap = 200 * 1024;
    Args a{};
    a.N = N;
    a.ncols = ncols;
    a.Q = Q;
    a.ldq = ldq;
    a.w = w;
    a.partial = fs.partial;
    a.PS = ncols + 2;
    a.h1 = fs.h1;
    a.h2 = fs.h2;
    a.h3 = fs.h3;
    a.flags = fs.flags;
    a.epoch = fs.epoch;
    a.gate = fs.gate;
    a.gate_want = fs.gate_want;
    a.ctrl = ctrl;
    a.t_entry = t_entry;
    a.check = check;
    a.pre_h = pre_h;
    // a column of this basis left pending by the previous (streaming) call on
    // this side is formed by the streaming kernel's first sweep: go there (the
    // automatic choice is monotone in the basis size, so it would anyway)
    const bool pending = fs.defer_st && fs.maybe_pending;
    auto flush_pending = [&]() {
        if (pending) flush_deferred(N, const_cast<double *>(Q), ldq, fs.defer_st, nsm, s);
    };
    if (fs.deferred) *fs.deferred = false;
    // small bases: one thread-block cluster, DSMEM reductions (measured: 12.7 vs
    // 17.2 us per call at config 1 (1.2 MB); slower than the Q-resident kernel
    // at 6 MB, the config 2 V side)
    if ((pol == 0 || pol == 5) && !pending) {
        const size_t cl_max = (size_t)2 << 20;
        const int C = 16;
        if (ncols <= 64 && (pol == 5 || (size_t)N * (size_t)std::max(ncols, 1) * 8 <= cl_max)) {
            // narrow bases: the latency-arranged cluster kernel
            const int64_t rpb = (N + C - 1) / C;
            const int PS = ncols + 2;
            const size_t smem = ((size_t)rpb + PS + 16 * (size_t)PS + 3 * (size_t)C * PS +
                                 (size_t)ncols * (size_t)(rpb | 1)) * sizeof(double);
            if (smem <= 200 * 1024) {
                CArgs ca{};
                ca.N = N;
                ca.ncols = ncols;
                ca.Q = Q;
                ca.ldq = ldq;
                ca.w = w;
                ca.ctrl = ctrl;
                ca.t_entry = t_entry;
                ca.check = check;
                ca.pre_h = pre_h;
                if (fs.pre) ca.pre = *fs.pre;
                ca.rpb = (int)rpb;
                ca.flags = fs.flags;
                ca.epoch = fs.epoch;
                ca.gate = fs.gate;
                ca.gate_want = fs.gate_want;
                auto kern = ncols <= 32 ? k_cgs2_cl<1> : k_cgs2_cl<2>;
                static bool attr[2] = {false, false};
                if (!attr[ncols > 32]) {
                    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                    attr[ncols > 32] = true;
                }
                if (launch_pdl(kern, dim3(C), dim3(kClThreads), smem, s, C, ca) == cudaSuccess) {
                    count_launch();
                    return true;
                }
                cudaGetLastError();
            }
        }
        const int64_t rpb = ((N + C - 1) / C + 1) / 2 * 2;  // even: 16-byte aligned Q segments
        const size_t smem0 = ((size_t)rpb + 4 * ((size_t)ncols + 2)) * sizeof(double);
        // the CTA's rows of Q staged in shared memory when they fit (bases <= 2 MB:
        // <= 128 KB per CTA) and ldq keeps them 16-byte aligned
        const bool qstage = ncols > 0 && (ldq % 2 == 0) && ((reinterpret_cast<uintptr_t>(Q) & 15) == 0) &&
                            smem0 + (size_t)ncols * rpb * sizeof(double) <= 200 * 1024;
        const size_t smem = smem0 + (qstage ? (size_t)ncols * rpb * sizeof(double) : 0);
        if ((pol == 5 || (size_t)N * (size_t)std::max(ncols, 1) * 8 <= cl_max) && smem <= 200 * 1024 &&
            ncols <= 1022) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_cgs2_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                cudaFuncSetAttribute(k_cgs2_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                attr = true;
            }
            CArgs ca{};
            ca.N = N;
            ca.ncols = ncols;
            ca.Q = Q;
            ca.ldq = ldq;
            ca.w = w;
            ca.ctrl = ctrl;
            ca.t_entry = t_entry;
            ca.check = check;
            ca.pre_h = pre_h;
            if (fs.pre) ca.pre = *fs.pre;
            ca.rpb = (int)rpb;
            ca.flags = fs.flags;
            ca.epoch = fs.epoch;
            ca.gate = fs.gate;
            ca.gate_want = fs.gate_want;
            ca.qstage = qstage ? 1 : 0;
            if (launch_pdl(k_cgs2_cluster, dim3(C), dim3(kClThreads), smem, s, C, ca) == cudaSuccess) {
                count_launch();
                return true;
            }
            cudaGetLastError();
        }
        if (pol == 5) return false;
    }
    // Q-resident mode: the CTA's rows of Q staged once in shared memory (1 CTA
    // per SM measured faster than 2: fewer CTAs in each grid barrier / reduction)
    if ((pol == 0 || pol == 2) && !pending) {
        const int nb = nsm;
        const int64_t rpb = (N + nb - 1) / nb;
        const size_t smem = ((size_t)ncols + 2 + rpb + (size_t)ncols * (rpb + 1) + std::max<int64_t>(256, rpb)) * sizeof(double);
        if (ncols > 0 && smem <= smem_cap && rpb >= 1) {
            a.rpb = (int)rpb;
            a.RT = 1;
            a.wsmem = 1;
            if (fs.pre) a.pre = *fs.pre;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_cgs2_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                attr = true;
            }
            int bps = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cgs2_fused<true>, kThreads, smem);
            if (bps >= 1) {
                const int grid = (int)std::min<int64_t>(nb, (N + rpb - 1) / rpb);
                void *args[] = {&a};
                if (cudaLaunchCooperativeKernel((void *)k_cgs2_fused<true>, grid, kThreads, args, smem, s) ==
                    cudaSuccess) {
                    count_launch();
                    return true;
                }
                cudaGetLastError();  // clear, fall through to the streaming kernel
            }
        }
        if (pol == 2) return false;
    }
    // streaming mode (tall bases): row tiles through shared memory; a pending
    // dense reduction is finished first (the tiles read w from HBM)
    if (fs.pre) split_reduce(N, *fs.pre, w, ctrl ? &ctrl->abort : nullptr, s);
    const bool aligned = (ldq % 2 == 0) && ((reinterpret_cast<uintptr_t>(Q) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    if (!aligned || ncols > 1024) {
        flush_pending();  // the caller's split sweeps need the column formed
        return false;
    }
    SArgs sa{};
    sa.N = N;
    sa.ncols = ncols;
    sa.Q = Q;
    sa.ldq = ldq;
    sa.w = w;
    sa.partial = fs.partial;
    sa.PS = ncols + 2;
    sa.h1 = fs.h1;
    sa.h2 = fs.h2;
    sa.h3 = fs.h3;
    sa.flags = fs.flags;
    sa.epoch = fs.epoch;
    sa.gate = fs.gate;
    sa.gate_want = fs.gate_want;
    sa.ctrl = ctrl;
    sa.t_entry = t_entry;
    sa.check = check;
    sa.pre_h = pre_h;
    sa.snake = 1;
    sa.phase = 0;
    if (pol == 4) {
        flush_pending();
        return tmap && launch_tma_any(*reinterpret_cast<const CUtensorMap *>(tmap), sa, nsm, s);
    }
    // cp.async register-blocked streaming (measured faster than the TMA variant
    // by 5-10 %); bases wider than its shared-memory ring (about
    // 860 columns) fall back to the split kernels
    if (fs.defer_st) {  // deferred second update
        sa.dst = fs.defer_st;
        sa.qw = const_cast<double *>(Q);
        sa.xs = fs.xs;
        sa.defer = (fs.xs && ncols > 0) ? 1 : 0;
    }
    if (!launch_stream2_any(sa, nsm, s)) {
        flush_pending();
        return false;
    }
    if (fs.deferred) *fs.deferred = sa.defer != 0;
    return true;
}

// Multi-GPU CGS2 (P > 1): the streaming kernel in three launches, split at its
// two reductions, with the cross-rank all-reduces of h1 and [h2; ||w'||^2]
// between them (SURVEY.md 8(e) collectives 2-3 / 5-6).  Each CTA reduction is
// finished on the device, so the all-reduce moves ncols (+1) doubles per rank.
// false: not applicable (caller uses the split sweeps).
bool cgs2_phased(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
                 const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nsm, cudaStream_t s,
                 Comm *comm, unsigned int *launches) {
    if (g_policy.cgs2 == 1) return false;
    const bool aligned = (ldq % 2 == 0) && ((reinterpret_cast<uintptr_t>(Q) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    if (!aligned || N < 1) return false;
    if (ncols > 840) return false;  // wider than the streaming kernel's shared-memory ring
    SArgs sa{};
    sa.N = N;
    sa.ncols = ncols;
    sa.Q = Q;
    sa.ldq = ldq;
    sa.w = w;
    sa.partial = fs.partial;
    sa.PS = ncols + 2;
    sa.h1 = fs.h1;
    sa.h2 = fs.h2;
    sa.h3 = fs.h3;
    sa.flags = fs.flags;
    sa.gate = nullptr;
    sa.ctrl = ctrl;
    sa.t_entry = t_entry;
    sa.check = check;
    sa.snake = 1;
    auto launch = [&](int phase) {
        sa.phase = phase;
        sa.epoch = 16u * (++*launches);
        sa.pre_h = phase == 1 ? pre_h : nullptr;
        if (!launch_stream2_any(sa, nsm, s))
            throw CommError(SVDSC_ECUDA, "multi-GPU CGS2: streaming kernel launch failed");
    };
    if (ncols > 0) {
        launch(1);
        comm->allreduce_sum(fs.h1, (size_t)ncols, s);
    } else if (pre_h) {
        return false;
    }
    launch(2);
    comm->allreduce_sum(fs.h2, (size_t)ncols + 1, s);
    launch(3);
    return true;
}

namespace {
// a pending column formed outside the streaming kernel: (w' - Q h2) / beta
// (pass end, before a breakdown repair, or before a non-streaming CGS2 call)
__global__ void __launch_bounds__(256) k_flush_deferred(int64_t N, double *__restrict__ Q, int64_t ldq,
                                                        const DeferState *__restrict__ st) {
    if (!*(volatile const int *)&st->flag) return;
    const int pc = st->col;
    const double rb = st->rbeta;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        int j = 0;
        for (; j + 1 < pc; j += 2) {
            s0 = fma(Q[r + (int64_t)j * ldq], st->h[j], s0);
            s1 = fma(Q[r + (int64_t)(j + 1) * ldq], st->h[j + 1], s1);
        }
        if (j < pc) s0 = fma(Q[r + (int64_t)j * ldq], st->h[j], s0);
        Q[r + (int64_t)pc * ldq] = (Q[r + (int64_t)pc * ldq] - (s0 + s1)) * rb;
    }
}
__global__ void k_flush_clear(DeferState *st) { st->flag = 0; }
}  // namespace

void flush_deferred(int64_t N, double *Q, int64_t ldq, DeferState *st, int nsm, cudaStream_t s) {
    if (N > 0) {
        k_flush_deferred<<<nsm * 8, 256, 0, s>>>(N, Q, ldq, st);
        count_launch();
    }
    k_flush_clear<<<1, 1, 0, s>>>(st);
    count_launch();
}

size_t peer_mailbox_bytes(int P, int PS) { return kPeerHdrBytes + (size_t)2 * P * PS * sizeof(double); }

namespace {
SArgs peer_sargs(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
                 const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, const PeerArgs *peer) {
    SArgs sa{};
    sa.N = N;
    sa.ncols = ncols;
    sa.Q = Q;
    sa.ldq = ldq;
    sa.w = w;
    sa.partial = fs.partial;
    sa.PS = ncols + 2;
    sa.h1 = fs.h1;
    sa.h2 = fs.h2;
    sa.h3 = fs.h3;
    sa.flags = fs.flags;
    sa.epoch = fs.epoch;
    sa.gate = nullptr;
    sa.ctrl = ctrl;
    sa.t_entry = t_entry;
    sa.check = check;
    sa.pre_h = pre_h;
    sa.snake = 1;
    sa.phase = 0;
    sa.peer = peer;
    return sa;
}
bool peer_applicable(int ncols, const double *Q, int64_t ldq, const double *w) {
    if (g_policy.cgs2 == 1) return false;
    const bool aligned = (ldq % 2 == 0) && ((reinterpret_cast<uintptr_t>(Q) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    return aligned && ncols <= 840;  // wider than the streaming kernel's shared-memory ring
}
}  // namespace

// Multi-GPU CGS2 over peer memory: one launch per
// re-orthogonalization; the h1 and [h2; ||w'||^2] all-reduces (and the rare
// explicit norm, reading G3) run inside the kernel as one-shot pushes into the
// ranks' mailboxes -- no NCCL call, no kernel boundary, no host round trip.
bool cgs2_peer(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
               const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nb, cudaStream_t s,
               const PeerArgs *peer) {
    // the deferred second update (reading G5) works per rank: the pending
    // column is formed from local rows with the (replicated) h2 and 1/beta
    const bool pending = fs.defer_st && fs.maybe_pending;
    if (fs.deferred) *fs.deferred = false;
    if (!peer || N < 1 || !peer_applicable(ncols, Q, ldq, w)) {
        if (pending) flush_deferred(N, const_cast<double *>(Q), ldq, fs.defer_st, nb, s);
        return false;
    }
    SArgs sa = peer_sargs(N, ncols, Q, ldq, w, pre_h, fs, ctrl, t_entry, check, peer);
    if (fs.defer_st) {
        sa.dst = fs.defer_st;
        sa.qw = const_cast<double *>(Q);
        sa.xs = fs.xs;
        sa.defer = (fs.xs && ncols > 0) ? 1 : 0;
    }
    if (!launch_stream2p_any(&sa, 1, nb, nullptr, s)) {
        if (pending) flush_deferred(N, const_cast<double *>(Q), ldq, fs.defer_st, nb, s);
        return false;
    }
    if (fs.deferred) *fs.deferred = sa.defer != 0;
    return true;
}

size_t cgs2_peer_emulate_grp_bytes(int P) { return (size_t)P * sizeof(SArgs); }

bool cgs2_peer_emulate(int P, int ncols, const PeerEmuRank *ranks, int nb, void *grp_dev, cudaStream_t s) {
    if (P < 1 || P > kMaxPeers) return false;
    std::vector<SArgs> ga((size_t)P);
    for (int g = 0; g < P; g++) {
        const PeerEmuRank &r = ranks[g];
        if (r.N < 1 || !peer_applicable(ncols, r.Q, r.ldq, r.w)) return false;
        ga[g] = peer_sargs(r.N, ncols, r.Q, r.ldq, r.w, nullptr, r.fs, r.ctrl, r.t_entry, 0, r.peer);
    }
    return launch_stream2p_any(ga.data(), P, nb, grp_dev, s);
}

namespace {
// one CTA, one exchange of the peer protocol (the CGS2 kernel's, with nb = 1)
__global__ void k_peer_check(const PeerArgs *pa, int n, double *out, Ctrl *ctrl) {
    const int P = pa->P, PS = pa->PS;
    const unsigned int rs = *(volatile const unsigned int *)pa->seq + 1u;
    const int par = (int)(rs & 1u);
    const int64_t slot = ((int64_t)par * P + pa->rank) * PS;
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        for (int q = 0; q < P; q++) __stcg(pa->mbox_peer[q] + slot + j, (double)(pa->rank + 1) * (double)(j + 1));
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int q = 0; q < P; q++) red_release_sys_add(pa->ctr_peer[q] + par, 1u);
        const unsigned int target = ((rs + 1u) >> 1) * (unsigned)P;  // one CTA per rank
        const long long t0 = clock64();
        while (ld_acquire_sys(pa->ctr + par) < target) {
            if (clock64() - t0 > kPeerTimeoutCycles) {
                ctrl->abort_kind = 2;
                break;
            }
        }
        __threadfence();
    }
    __syncthreads();
    const double *sl = pa->mbox + (int64_t)par * P * PS;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double s = __ldcg(sl + j);
        for (int q = 1; q < P; q++) s += __ldcg(sl + (int64_t)q * PS + j);
        out[j] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *pa->seq = rs;
}
}  // namespace

// one arrival per rank instead of PeerArgs::expect: the caller runs it on
// freshly reset counters (peer_reset + a collective), and the next solve resets
// them again before its CGS2 kernels count P x nb arrivals per exchange
void peer_check(const PeerArgs *peer, int n, double *out, Ctrl *ctrl, cudaStream_t s) {
    k_peer_check<<<1, 256, 0, s>>>(peer, n, out, ctrl);
    count_launch();
}

}  // namespace svdsc
