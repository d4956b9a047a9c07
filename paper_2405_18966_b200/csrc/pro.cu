// pro.cu -- partial re-orthogonalization decisions (opts.reorth = 1).
//
// SURVEY.md 8(f4); reading Q20.  The paper names this class of
// method (PROPACK lansvd) without its rules; they are the
// omega recurrence of Simon / Larsen restated for this algorithm's T (upper
// bidiagonal in the first pass, the arrow of Alg. 2 step 9 after a restart):
// with A v_l = sum_{p<=l} T(p,l) u_p and A^T u_l = sum_{p>=l} T(l,p) v_p,
//   V side (v_i from w):  nu_l  <- (sum_{p<=l} T(p,l) mu_p - alpha nu_l  +- eps1) / ||w||
//   U side (u_i from z):  mu_l  <- (sum_{l<=p<=i} T(l,p) nu_p - beta mu_l +- eps1) / ||z||
// eps1 = eps * (largest column 1-norm of the completed columns of T).  The new
// vector is re-orthogonalized (the full fused CGS2 kernel runs) iff some
// |estimate| > sqrt(eps), its norm is 0, or the previous vector of the side
// was re-orthogonalized because of its estimate; its row is then reset to eps.
//
// Per half-step: k_pro_partial (grid, ||x||^2 partials in a fixed order) and
// k_pro_decide (one CTA: the norm, the row update, the decision) write
// ctrl->pro_gate; the two fused CGS2 launches that follow are gated on it
// (full re-orthogonalization if 1, normalization only if 0).  All kernels
// are no-ops while a breakdown abort is pending (replay-safe, Ctrl::abort).
//
// The arithmetic of the row update is written with explicit _rn operations in
// the oracle's order (no FMA contraction), so that given the same T, rows and
// norm both sides take bit-identical decisions.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace svdsc {
namespace {

constexpr double kEps = 2.220446049250313e-16;        // 2^-52
constexpr double kDelta = 1.4901161193847656e-08;     // sqrt(2^-52) = 2^-26
constexpr int kDecThreads = 512;

__device__ __forceinline__ double tsum_ordered(double x, double a, double b) {
    return __dadd_rn(x, __dmul_rn(a, b));
}

__global__ void __launch_bounds__(256) k_pro_partial(int64_t N, const double *__restrict__ x, double *part,
                                                    const int *abort) {
    if (*(volatile const int *)abort) return;
    __shared__ double sh[32];
    const int64_t chunk = (N + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(N, r0 + chunk);
    double s = 0.0;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) s = fma(x[r], x[r], s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = s;
    __syncthreads();
    if (wid == 0) {
        double v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) part[blockIdx.x] = v;
    }
}

__device__ double dec_sum(double v, double *sh) {  // fixed tree over the CTA
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    for (int q = 0; q < kDecThreads / 32; q++) r += sh[q];
    return r;
}

__device__ double dec_max(double v, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    for (int q = 0; q < kDecThreads / 32; q++) r = fmax(r, sh[q]);
    return r;
}

// side 0: V side of step i (row nu of v_i); side 1: U side (row mu of u_i).
// kr: the arrow column of T (k after a restart), -1 in the first pass.
__global__ void __launch_bounds__(kDecThreads) k_pro_decide(int side, int i, int kr, const double *__restrict__ T,
                                                            int ldt, const double *__restrict__ part, int nparts,
                                                            double *mu, double *nu, Ctrl *ctrl) {
    if (*(volatile const int *)&ctrl->abort) return;
    __shared__ double sh[32];
    __shared__ int sviol;
    extern __shared__ double sarrow[];  // the arrow column T(0:kr, kr) and mu(0:kr), staged in parallel
    const int tid = threadIdx.x;
    auto Tm = [&](int p, int l) { return T[p + (int64_t)l * ldt]; };
    if (kr >= 0) {
        for (int p = tid; p <= kr; p += kDecThreads) {
            sarrow[p] = Tm(p, kr);
            sarrow[kr + 1 + p] = mu[p];
        }
        __syncthreads();
    }
    // ||x||: the partials in a fixed order
    double ps = 0.0;
    for (int b = tid; b < nparts; b += kDecThreads) ps += part[b];
    const double nrm = sqrt(dec_sum(ps, sh));
    // eps1 = eps * max column 1-norm of T(:, 0:i-1), summed in the oracle's order
    double am = 0.0;
    for (int l = tid; l < i; l += kDecThreads) {
        double c;
        if (kr >= 0 && l == kr) {
            c = 0.0;
            for (int p = 0; p <= kr; p++) c = __dadd_rn(c, fabs(sarrow[p]));
        } else if (kr >= 0 && l < kr) {
            c = fabs(Tm(l, l));
        } else {
            c = (l >= 1) ? __dadd_rn(fabs(Tm(l - 1, l)), fabs(Tm(l, l))) : fabs(Tm(l, l));
        }
        am = fmax(am, c);
    }
    const double eps1 = __dmul_rn(kEps, dec_max(am, sh));
    double *row = side == 0 ? nu : mu;
    double vmax = 0.0;
    if (side == 0) {
        const double alpha = Tm(i - 1, i - 1);
        for (int l = tid; l < i; l += kDecThreads) {
            double x = 0.0;  // column l of T against mu
            if (kr >= 0 && l == kr) {
                for (int p = 0; p <= kr; p++) x = tsum_ordered(x, sarrow[p], sarrow[kr + 1 + p]);
            } else if (kr >= 0 && l < kr) {
                x = tsum_ordered(x, Tm(l, l), mu[l]);
            } else {
                if (l >= 1) x = tsum_ordered(x, Tm(l - 1, l), mu[l - 1]);
                x = tsum_ordered(x, Tm(l, l), mu[l]);
            }
            x = __dsub_rn(x, __dmul_rn(alpha, nu[l]));
            x = __dadd_rn(x, x < 0.0 ? -eps1 : eps1);
            const double r = __ddiv_rn(x, nrm);
            nu[l] = r;
            vmax = (fabs(r) <= kDelta) ? vmax : 1.0;  // NaN counts as a violation
        }
    } else {
        const double beta = Tm(i - 1, i);
        for (int l = tid; l < i; l += kDecThreads) {
            double y = 0.0;  // row l of T against nu (nu[i] = 1)
            if (kr >= 0 && l < kr) {
                y = tsum_ordered(y, Tm(l, l), nu[l]);
                y = tsum_ordered(y, Tm(l, kr), nu[kr]);
            } else {
                y = tsum_ordered(y, Tm(l, l), nu[l]);
                y = tsum_ordered(y, Tm(l, l + 1), nu[l + 1]);
            }
            y = __dsub_rn(y, __dmul_rn(beta, mu[l]));
            y = __dadd_rn(y, y < 0.0 ? -eps1 : eps1);
            const double r = __ddiv_rn(y, nrm);
            mu[l] = r;
            vmax = (fabs(r) <= kDelta) ? vmax : 1.0;
        }
    }
    const bool viol = dec_max(vmax, sh) > 0.0 || !(nrm > 0.0);
    __shared__ int sforce;
    if (tid == 0) {
        sviol = viol;
        sforce = ctrl->pro_force[side];
    }
    __syncthreads();
    const int force = sforce;
    const bool reo = sviol || force;
    if (reo)
        for (int l = tid; l < i; l += kDecThreads) row[l] = kEps;
    if (tid == 0) {
        row[i] = 1.0;
        ctrl->pro_force[side] = (sviol && !force) ? 1 : 0;
        ctrl->pro_gate = reo ? 1 : 0;
        if (reo) ctrl->pro_reorths++;
    }
}

// after the restart: nu_j = sum_l nu_l Vh(l, j) (v_{k+1} = v_{t+1} against the
// Ritz vectors V Vh(:, 0:k-1)); u_{k+1} was re-orthogonalized in full
__global__ void __launch_bounds__(256) k_pro_restart(int t, int k, const double *__restrict__ Vh, int ldvh,
                                                    double *mu, double *nu, Ctrl *ctrl) {
    extern __shared__ double tmp[];
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        double s = 0.0;
        for (int l = 0; l < t; l++) s = tsum_ordered(s, nu[l], Vh[l + (int64_t)j * ldvh]);
        tmp[j] = s;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        nu[j] = tmp[j];
        mu[j] = kEps;
    }
    if (threadIdx.x == 0) {
        nu[k] = 1.0;
        mu[k] = 1.0;
        ctrl->pro_force[0] = ctrl->pro_force[1] = 0;
    }
}

__global__ void k_pro_init(int len, double *mu, double *nu) {
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
        mu[j] = j == 0 ? 1.0 : 0.0;
        nu[j] = j == 0 ? 1.0 : 0.0;
    }
}

}  // namespace

void pro_init(int t, double *mu, double *nu, cudaStream_t s) {
    k_pro_init<<<1, 256, 0, s>>>(t + 2, mu, nu);
    count_launch();
}

void pro_decide(int side, int64_t N, const double *x, int i, int kr, const double *T, int ldt, double *mu,
                double *nu, double *part, Ctrl *ctrl, int nsm, cudaStream_t s) {
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(nsm, (N + 255) / 256));
    k_pro_partial<<<nb, 256, 0, s>>>(N, x, part, &ctrl->abort);
    count_launch();
    const size_t smem = kr >= 0 ? 2 * (size_t)(kr + 1) * sizeof(double) : 0;
    k_pro_decide<<<1, kDecThreads, smem, s>>>(side, i, kr, T, ldt, part, nb, mu, nu, ctrl);
    count_launch();
}

void pro_restart(int t, int k, const double *Vh, int ldvh, double *mu, double *nu, Ctrl *ctrl, cudaStream_t s) {
    k_pro_restart<<<1, 256, (size_t)std::max(k, 1) * sizeof(double), s>>>(t, k, Vh, ldvh, mu, nu, ctrl);
    count_launch();
}

}  // namespace svdsc
