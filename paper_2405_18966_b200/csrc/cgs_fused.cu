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
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

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

// sense-free generation barrier over all CTAs of a cooperative launch
__device__ __forceinline__ void grid_barrier(unsigned int *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (ld_acquire(bar + 1) == gen) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

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
    unsigned int *bar;
    Ctrl *ctrl;
    double *t_entry;
    int check;
    const double *pre_h;  // optional w -= Q pre_h before the passes (Alg. 2 step 10)
    int rpb;              // rows per CTA
    int RT;               // row tile of phase B (streaming mode)
    int wsmem;            // keep the CTA's w rows in shared memory
};

// out[j] = sum_b partial[b][j] for the columns owned by this CTA
__device__ void reduce_cols(const Args &a, int ncols_tot, double *out, double *sh) {
    const int nb = gridDim.x;
    for (int j = blockIdx.x; j < ncols_tot; j += nb) {
        double s = 0.0;
        for (int t = threadIdx.x; t < nb; t += blockDim.x) s += __ldcg(a.partial + (int64_t)t * a.PS + j);
        s = block_sum_all(s, sh);
        if (threadIdx.x == 0) out[j] = s;
    }
}

template <bool QS>
__device__ __forceinline__ double qval(const Args &a, const double *qsh, int ldqs, int64_t r0, int i, int j) {
    if (QS) return qsh[j * ldqs + i];
    return __ldg(a.Q + r0 + i + (int64_t)j * a.ldq);
}

template <bool QS>
__global__ void __launch_bounds__(256) k_cgs2_fused(Args a) {
    if (*(volatile int *)&a.ctrl->abort) return;  // uniform over the grid
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
    double *part = qsh + (QS ? 0 : (int64_t)ncols * LDT);  // 256
    double *wpt = part + 256;                               // RT
    double *wv = a.wsmem ? wsh : (a.w + r0);  // generic pointer to this CTA's rows of w

    if (a.wsmem)
        for (int i = tid; i < nr; i += blockDim.x) wsh[i] = a.w[r0 + i];
    if (QS) {
        for (int idx = tid; idx < ncols * nr; idx += blockDim.x) {
            const int j = idx / nr, i = idx - j * nr;
            qsh[j * ldqs + i] = a.Q[r0 + i + (int64_t)j * a.ldq];
        }
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

    double nrm_wp = 0.0;  // ||w'||^2 partial (thread-local)
    if (ncols > 0) {
        // ---------------- phase A: partial h1 ----------------
        if (QS) {
            for (int j = wid; j < ncols; j += 8) {
                double s = 0.0;
                for (int i = lane; i < nr; i += 32) s = fma(qsh[j * ldqs + i], wv[i], s);
                s = warp_sum(s);
                if (lane == 0) a.partial[(int64_t)blockIdx.x * a.PS + j] = s;
            }
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
        grid_barrier(a.bar);
        reduce_cols(a, ncols, a.h1, sh);
        grid_barrier(a.bar);
        for (int j = tid; j < ncols; j += blockDim.x) hs[j] = __ldcg(a.h1 + j);
        __syncthreads();

        // ---------------- phase B: w' = w - Q h1, partial h2, ||w'||^2 ----------------
        if (QS) {
            for (int i = tid; i < nr; i += blockDim.x) {
                double s = 0.0;
                for (int j = 0; j < ncols; j++) s = fma(qsh[j * ldqs + i], hs[j], s);
                const double v = wv[i] - s;
                wv[i] = v;
                nrm_wp = fma(v, v, nrm_wp);
            }
            __syncthreads();
            for (int j = wid; j < ncols; j += 8) {
                double s = 0.0;
                for (int i = lane; i < nr; i += 32) s = fma(qsh[j * ldqs + i], wv[i], s);
                s = warp_sum(s);
                if (lane == 0) a.partial[(int64_t)blockIdx.x * a.PS + j] = s;
            }
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
        grid_barrier(a.bar);
        reduce_cols(a, ncols + 1, a.h2, sh);
        grid_barrier(a.bar);
        for (int j = tid; j <= ncols; j += blockDim.x) hs[j] = __ldcg(a.h2 + j);
        __syncthreads();
    } else {
        // plain norm: ||w||^2 into hs[0] (ncols == 0)
        for (int i = tid; i < nr; i += blockDim.x) nrm_wp = fma(wv[i], wv[i], nrm_wp);
        const double bn = block_sum_all(nrm_wp, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS] = bn;
        grid_barrier(a.bar);
        reduce_cols(a, 1, a.h2, sh);
        grid_barrier(a.bar);
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
        for (int i = tid; i < nr; i += blockDim.x) {
            double s = 0.0;
#pragma unroll 8
            for (int j = 0; j < ncols; j++) s = fma(qval<QS>(a, qsh, ldqs, r0, i, j), hs[j], s);
            const double v = wv[i] - s;
            wv[i] = v;
            nrm2 = fma(v, v, nrm2);
        }
    }
    __syncthreads();
    if (!pyth) {  // explicit norm (uniform branch: every CTA sees the same hs)
        const double bn = block_sum_all(nrm2, sh);
        if (tid == 0) a.partial[(int64_t)blockIdx.x * a.PS] = bn;
        grid_barrier(a.bar);
        reduce_cols(a, 1, a.h3, sh);
        grid_barrier(a.bar);
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
    if (bd) return;
    for (int i = tid; i < nr; i += blockDim.x) a.w[r0 + i] = wv[i] / beta;
}

}  // namespace

// returns false if the fused path cannot be used (caller falls back)
bool cgs2_fused(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *pre_h,
                const FusedScratch &fs, Ctrl *ctrl, double *t_entry, int check, int nsm, cudaStream_t s) {
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
    a.bar = fs.bar;
    a.ctrl = ctrl;
    a.t_entry = t_entry;
    a.check = check;
    a.pre_h = pre_h;
    // try Q-resident mode: 2 CTAs per SM, then 1
    for (int per_sm = 2; per_sm >= 1; per_sm--) {
        const int nb = nsm * per_sm;
        const int64_t rpb = (N + nb - 1) / nb;
        const size_t smem = ((size_t)ncols + 2 + rpb + (size_t)ncols * (rpb + 1)) * sizeof(double);
        if (ncols > 0 && smem * per_sm <= 220 * 1024 && smem <= smem_cap && rpb >= 1) {
            a.rpb = (int)rpb;
            a.RT = 1;
            a.wsmem = 1;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_cgs2_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                attr = true;
            }
            int bps = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cgs2_fused<true>, kThreads, smem);
            if (bps < per_sm) continue;
            const int grid = (int)std::min<int64_t>(nb, (N + rpb - 1) / rpb);
            void *args[] = {&a};
            if (cudaLaunchCooperativeKernel((void *)k_cgs2_fused<true>, grid, kThreads, args, smem, s) != cudaSuccess)
                return false;
            count_launch();
            return true;
        }
    }
    // streaming mode
    int RT = 64;
    while (RT > 8 && (size_t)ncols * (RT + 1) * 8 > 80 * 1024) RT >>= 1;
    const int per_sm = 2;
    const int nb = nsm * per_sm;
    int64_t rpb = (N + nb - 1) / nb;
    const int wsmem = rpb <= 2048 ? 1 : 0;
    const size_t smem = ((size_t)ncols + 2 + (wsmem ? rpb : 0) + (size_t)ncols * (RT + 1) + 256 + RT) * sizeof(double);
    if (smem > smem_cap || ncols > 1024) return false;
    a.rpb = (int)rpb;
    a.RT = RT;
    a.wsmem = wsmem;
    static bool attr2 = false;
    if (!attr2) {
        cudaFuncSetAttribute(k_cgs2_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr2 = true;
    }
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cgs2_fused<false>, kThreads, smem);
    if (bps < 1) return false;
    const int grid = (int)std::min<int64_t>((int64_t)nsm * std::min(bps, per_sm), (N + rpb - 1) / rpb);
    if ((int64_t)grid * rpb < N) {
        // fewer CTAs than planned: recompute rows per CTA
        rpb = (N + grid - 1) / grid;
        a.rpb = (int)rpb;
        a.wsmem = 0;
    }
    void *args[] = {&a};
    if (cudaLaunchCooperativeKernel((void *)k_cgs2_fused<false>, grid, kThreads, args, smem, s) != cudaSuccess)
        return false;
    count_launch();
    return true;
}

}  // namespace svdsc
