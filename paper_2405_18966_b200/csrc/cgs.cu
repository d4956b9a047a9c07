// cgs.cu -- full re-orthogonalization of each new Lanczos vector
// (w <- (I - Q Q^T) w against all stored basis vectors), done as
// two classical Gram-Schmidt passes (reading Q1), and the norms that
// give the bidiagonal entries (Alg. 1 lines 6 and 8).
// SURVEY.md 8(a) rows a2-a4 (V side) and a6 (U side).
//
// Three sweeps over the tall-skinny basis Q (N x ncols, column-major):
//   p1:  h1 = Q^T w                                    (one read of Q)
//   p2:  w' = w - Q h1 (in place);  h2 = Q^T w'        (one read of Q: each CTA
//        stages a row tile of Q in shared memory and uses it twice)
//   p3:  w'' = w' - Q h2 (in place);  ||w''||^2         (one read of Q)
// then normalize: beta = ||w''||, breakdown test, T entry, w'' / beta.
// Every reduction over rows is two-level: per-CTA partials in a fixed-shape
// tree, then the last CTA to finish sums the partials in block order -- the
// result is bitwise reproducible run to run.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace svdsc {
namespace {

__device__ __forceinline__ bool aborted(const int *abort) {
    return abort != nullptr && *(volatile const int *)abort != 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// true on every thread of the last CTA to arrive (the counter is reset by it)
__device__ __forceinline__ bool last_block(unsigned int *cnt) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(cnt, 1u) == gridDim.x - 1);
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// out[j] = sum_b partial[j*pstride + b], b = 0..nb-1, warp per column, fixed order
__device__ __forceinline__ void reduce_partials(const double *partial, int pstride, int nb, int ncols,
                                                double *out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = w; j < ncols; j += nw) {
        double s = 0.0;
        for (int b = lane; b < nb; b += 32) s += __ldcg(partial + (int64_t)j * pstride + b);
        s = warp_sum(s);
        if (lane == 0) out[j] = s;
    }
}

__device__ __forceinline__ double block_sum(double v, double *sh /* >= 32 */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += sh[i];
    return s;  // thread 0
}

constexpr int kTile = 16;  // columns per register tile in p1

// Transpose-reduce: lane l holds acc[0..15]; returns (on every lane) the sum over
// the 32 lanes of acc[l & 15].  4 butterfly stages + one half-warp swap.
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

// p1: partial h1 over this CTA's contiguous row range
__global__ void __launch_bounds__(256) k_cgs_p1(int64_t N, int ncols, const double *__restrict__ Q, int64_t ldq,
                                                const double *__restrict__ w, double *partial, int pstride,
                                                double *out, unsigned int *cnt, const int *abort) {
    if (aborted(abort)) return;
    __shared__ double sred[8][kTile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t rpb = (N + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * rpb, r1 = min(N, r0 + rpb);
    for (int j0 = 0; j0 < ncols; j0 += kTile) {
        const int nc = min(kTile, ncols - j0);
        double acc[kTile];
#pragma unroll
        for (int q = 0; q < kTile; q++) acc[q] = 0.0;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
            const double wr = w[r];
            const double *qp = Q + r + (int64_t)j0 * ldq;
#pragma unroll
            for (int q = 0; q < kTile; q++)
                if (q < nc) acc[q] = fma(qp[(int64_t)q * ldq], wr, acc[q]);
        }
        const double v = butterfly16(acc, lane);
        if (lane < kTile) sred[wid][lane] = v;
        __syncthreads();
        if (threadIdx.x < nc) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < 8; q++) s += sred[q][threadIdx.x];
            partial[(int64_t)(j0 + threadIdx.x) * pstride + blockIdx.x] = s;
        }
        __syncthreads();
    }
    if (last_block(cnt)) {
        reduce_partials(partial, pstride, gridDim.x, ncols, out);
        if (threadIdx.x == 0) *cnt = 0;
    }
}

// p2: w' = w - Q h1 (in place), partial h2 = Q^T w', ||w'||^2 -> out[ncols]
__global__ void __launch_bounds__(256) k_cgs_p2(int64_t N, int ncols, const double *__restrict__ Q, int64_t ldq,
                                                double *w, const double *__restrict__ h1, double *partial,
                                                int pstride, double *out, unsigned int *cnt, const int *abort,
                                                int RT) {
    if (aborted(abort)) return;
    extern __shared__ double sm[];
    const int LDT = RT + 1;
    double *tile = sm;                        // ncols x LDT
    double *hs = tile + (int64_t)ncols * LDT; // ncols
    double *wp = hs + ncols;                  // RT
    double *part = wp + RT;                   // 256
    __shared__ double sh[32];
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) hs[j] = h1[j];
    const int P = blockDim.x / RT;
    const int rr = threadIdx.x % RT, pp = threadIdx.x / RT;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // columns threadIdx.x + 256 q (ncols <= 1024)
    double nrm = 0.0;
    const int64_t ntiles = (N + RT - 1) / RT;
    __syncthreads();
    for (int64_t tI = blockIdx.x; tI < ntiles; tI += gridDim.x) {
        const int64_t r0 = tI * RT;
        const int nr = (int)min((int64_t)RT, N - r0);
        for (int idx = threadIdx.x; idx < ncols * RT; idx += blockDim.x) {
            const int j = idx / RT, q = idx - j * RT;
            tile[j * LDT + q] = (q < nr) ? Q[r0 + q + (int64_t)j * ldq] : 0.0;
        }
        __syncthreads();
        double s = 0.0;
        for (int j = pp; j < ncols; j += P) s = fma(tile[j * LDT + rr], hs[j], s);
        part[pp * RT + rr] = s;
        __syncthreads();
        if (threadIdx.x < RT) {
            double tsum = 0.0;
            for (int q = 0; q < P; q++) tsum += part[q * RT + threadIdx.x];
            double v = 0.0;
            if (threadIdx.x < nr) {
                v = w[r0 + threadIdx.x] - tsum;
                w[r0 + threadIdx.x] = v;
                nrm = fma(v, v, nrm);
            }
            wp[threadIdx.x] = v;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int j = threadIdx.x + 256 * q;
            if (j < ncols) {
                double a = acc[q];
                const double *tj = tile + j * LDT;
                for (int k = 0; k < RT; k++) a = fma(tj[k], wp[k], a);
                acc[q] = a;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int j = threadIdx.x + 256 * q;
        if (j < ncols) partial[(int64_t)j * pstride + blockIdx.x] = acc[q];
    }
    const double bn = block_sum(nrm, sh);
    if (threadIdx.x == 0) partial[(int64_t)ncols * pstride + blockIdx.x] = bn;
    if (last_block(cnt)) {
        reduce_partials(partial, pstride, gridDim.x, ncols + 1, out);
        if (threadIdx.x == 0) *cnt = 0;
    }
}

// p3: w <- w - Q h (in place); ||w||^2 -> out[0].  ncols may be 0 (plain norm).
__global__ void __launch_bounds__(256) k_cgs_p3(int64_t N, int ncols, const double *__restrict__ Q, int64_t ldq,
                                                double *w, const double *__restrict__ h, double *partial,
                                                int pstride, double *out, unsigned int *cnt, const int *abort) {
    if (aborted(abort)) return;
    extern __shared__ double hs[];
    __shared__ double sh[32];
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) hs[j] = h[j];
    __syncthreads();
    double nrm = 0.0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        const double *qp = Q + r;
#pragma unroll 8
        for (int j = 0; j < ncols; j++) s = fma(qp[(int64_t)j * ldq], hs[j], s);
        const double v = w[r] - s;
        if (ncols > 0) w[r] = v;
        nrm = fma(v, v, nrm);
    }
    const double bn = block_sum(nrm, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = bn;
    if (last_block(cnt)) {
        reduce_partials(partial, pstride, gridDim.x, 1, out);
        if (threadIdx.x == 0) *cnt = 0;
    }
}

__global__ void k_normalize(int64_t N, double *w, const double *nrm2, Ctrl *ctrl, double *t_entry, int check,
                            int force) {
    if (!force && *(volatile int *)&ctrl->abort) return;
    const double nv = sqrt(*nrm2);
    const double amax = ctrl->amax[check & 1];
    const double thr = 1e-14 * fmax(amax, 1.0);
    const bool bd = !force && !(nv > thr);
    if (blockIdx.x == 0 && threadIdx.x == 0 && !force) {
        if (bd) {
            *t_entry = 0.0;
            ctrl->amax[(check + 1) & 1] = amax;
            ctrl->abort_check = check;
            __threadfence();
            ctrl->abort = 1;
        } else {
            *t_entry = nv;
            ctrl->amax[(check + 1) & 1] = fmax(amax, nv);
        }
    }
    if (bd) return;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x)
        w[r] = w[r] / nv;
}

// SplitMix64 finalizer, same constants as the documented definition (Q7)
__device__ __forceinline__ uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_breakdown_vec(int64_t N, int64_t off, double *w, uint64_t seed, uint64_t stream) {
    const uint64_t key = sm64(seed ^ sm64(stream * 0xD1B54A32D192ED03ull + 1ull));
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z = sm64(key + (uint64_t)(r + off) * 0x9E3779B97F4A7C15ull);
        w[r] = (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
    }
}

__global__ void k_random_start(int64_t N, int64_t off, double *w, uint64_t seed) {
    const uint64_t key = sm64(seed ^ 0x5851F42D4C957F2Dull);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z1 = sm64(key + (uint64_t)(2 * (r + off)) * 0x9E3779B97F4A7C15ull);
        const uint64_t z2 = sm64(key + (uint64_t)(2 * (r + off) + 1) * 0x9E3779B97F4A7C15ull);
        double u1 = ((double)(z1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        double u2 = (double)(z2 >> 11) * (1.0 / 9007199254740992.0);
        w[r] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    }
}

__global__ void k_axpy(int64_t N, double *y, const double *c_dev, const double *x, const int *abort) {
    if (aborted(abort)) return;
    const double c = *c_dev;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x)
        y[r] -= c * x[r];
}

int grid_rows(int64_t N, int nsm) {
    int64_t g = (N + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)nsm * 8));
}

}  // namespace

int cgs_blocks(int64_t N, int nsm) {
    // >= 4 rows per thread; a multiple of the SM count when the basis is tall
    const int64_t per_sm = (N + (int64_t)nsm * 1024 - 1) / ((int64_t)nsm * 1024);
    if (per_sm >= 1) return nsm * (int)std::min<int64_t>(per_sm, 4);
    return (int)std::max<int64_t>(1, (N + 1023) / 1024);
}

void cgs_p1(int64_t N, int ncols, const double *Q, int64_t ldq, const double *w, const RedBuf &r, const int *abort,
            int nsm, cudaStream_t s) {
    const int nb = std::min(cgs_blocks(N, nsm), kMaxBlocks);
    k_cgs_p1<<<nb, 256, 0, s>>>(N, ncols, Q, ldq, w, r.partial, r.pstride, r.h1, r.cnt, abort);
    count_launch();
}

void cgs_p2(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const RedBuf &r, const int *abort,
            int nsm, cudaStream_t s) {
    // row tile RT: ncols x (RT+1) doubles of shared memory, ~<= 100 KB -> 2 CTAs/SM
    int RT = 64;
    while (RT > 8 && (size_t)ncols * (RT + 1) * 8 > 100 * 1024) RT >>= 1;
    const size_t smem = ((size_t)ncols * (RT + 1) + ncols + RT + 256) * sizeof(double);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_cgs_p2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    const int64_t ntiles = (N + RT - 1) / RT;
    int per_sm = std::max(1, (int)((220 * 1024) / std::max<size_t>(smem + 1024, 1)));
    per_sm = std::min(per_sm, 8);
    const int nb = (int)std::min<int64_t>({ntiles, (int64_t)nsm * per_sm, (int64_t)kMaxBlocks});
    k_cgs_p2<<<nb, 256, smem, s>>>(N, ncols, Q, ldq, w, r.h1, r.partial, r.pstride, r.h2, r.cnt, abort, RT);
    count_launch();
}

void cgs_p3(int64_t N, int ncols, const double *Q, int64_t ldq, double *w, const double *h, const RedBuf &r,
            const int *abort, int nsm, cudaStream_t s) {
    const int nb = std::min(grid_rows(N, nsm), kMaxBlocks);
    k_cgs_p3<<<nb, 256, std::max(ncols, 1) * sizeof(double), s>>>(N, ncols, Q, ldq, w, h ? h : r.h2, r.partial,
                                                                    r.pstride, r.nrm, r.cnt, abort);
    count_launch();
}

void normalize(int64_t N, double *w, const RedBuf &r, Ctrl *ctrl, double *t_entry, int check, int force, int nsm,
               cudaStream_t s) {
    k_normalize<<<grid_rows(N, nsm), 256, 0, s>>>(N, w, r.nrm, ctrl, t_entry, check, force);
    count_launch();
}

void breakdown_vector(int64_t N, int64_t row_offset, double *w, uint64_t seed, uint64_t stream, cudaStream_t s) {
    k_breakdown_vec<<<grid_rows(N, 148), 256, 0, s>>>(N, row_offset, w, seed, stream);
    count_launch();
}

void random_start(int64_t N, int64_t row_offset, double *w, uint64_t seed, cudaStream_t s) {
    k_random_start<<<grid_rows(N, 148), 256, 0, s>>>(N, row_offset, w, seed);
    count_launch();
}

void axpy_dev(int64_t N, double *y, const double *c_dev, const double *x, const int *abort, cudaStream_t s) {
    k_axpy<<<grid_rows(N, 148), 256, 0, s>>>(N, y, c_dev, x, abort);
    count_launch();
}

}  // namespace svdsc
