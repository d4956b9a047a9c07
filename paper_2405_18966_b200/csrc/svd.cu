// svd.cu -- once-per-pass work of Alg. 2, on device:
//   a7  [Uh, Sh, Vh] = svd(T(1:t,1:t))           Alg. 2 step 4
//       res_j = |T(t,t+1) Uh(t,j)| / Sh(j,j)      Eq. (4); step 5
//   a8  rho = beta_t Uh(t,1:k)^T, T rebuilt       Alg. 2 step 9
//       Q(:,1:k) <- Q(:,1:t) W(:,1:k) in place    Alg. 2 step 8
//   a9  U_k, V_k assembly                         Alg. 2 step 16
// The paper calls LAPACKE_dgesvd.  After a restart T is
// "diagonal + one dense column + bidiagonal" (not bidiagonal), so
// the device SVD is a one-sided (Hestenes) Jacobi with a parallel round-robin
// pair ordering (t/2 independent rotations per round, one warp each), the
// rotation rule and threshold of the oracle, descending sort, and the sign
// rule of SPEC.md:158.  No CPU fallback.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace cg = cooperative_groups;

namespace svdsc {
namespace {

constexpr int kMaxP = 1024;

__device__ __forceinline__ bool aborted(const int *abort) {
    return abort != nullptr && *(volatile const int *)abort != 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// W = T(1:p,1:p), V = I, ctrl->svd_tiny = p eps ||T||_F (reading Q10b); one CTA,
// fixed-order reduction
__global__ void __launch_bounds__(1024) k_copy_T(int p, const double *__restrict__ T, int ldt, double *W, double *V,
                                                 Ctrl *ctrl, const int *abort) {
    if (aborted(abort)) return;
    __shared__ double sh[32];
    double s = 0.0;
    for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) {
        const int r = idx % p, c = idx / p;
        const double x = T[r + (int64_t)c * ldt];
        W[idx] = x;
        V[idx] = (r == c) ? 1.0 : 0.0;
        s = fma(x, x, s);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) tot += sh[i];
        ctrl->svd_tiny = (double)p * 2.220446049250313e-16 * sqrt(tot);
    }
}

// round-robin (circle method) pairing: round rnd in [0, pe-1), slot q in [0, pe/2)
__device__ __forceinline__ void rr_pair(int pe, int rnd, int q, int &a, int &b) {
    if (q == 0) {
        a = rnd;
        b = pe - 1;
    } else {
        a = (rnd + q) % (pe - 1);
        b = (rnd - q + (pe - 1)) % (pe - 1);
    }
    if (a > b) {
        int tmp = a;
        a = b;
        b = tmp;
    }
}

// One CTA, W (p x p) and V in global memory (L1/L2 resident).
__global__ void __launch_bounds__(1024) k_jacobi(int p, double *W, double *V, Ctrl *ctrl, const int *abort,
                                                 double ctol, int max_sweeps) {
    if (aborted(abort)) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int pe = p + (p & 1);
    const double tiny = *(volatile double *)&ctrl->svd_tiny;
    __shared__ int rotated;
    int sweep;
    bool conv = false;
    for (sweep = 1; sweep <= max_sweeps; sweep++) {
        if (threadIdx.x == 0) rotated = 0;
        __syncthreads();
        for (int rnd = 0; rnd < pe - 1; rnd++) {
            for (int q = wid; q < pe / 2; q += nw) {
                int a, b;
                rr_pair(pe, rnd, q, a, b);
                if (b >= p) continue;
                double *wa = W + (int64_t)a * p, *wb = W + (int64_t)b * p;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int r = lane; r < p; r += 32) {
                    const double x = wa[r], y = wb[r];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (!(sqrt(al) > tiny) || !(sqrt(be) > tiny)) continue;
                if (fabs(ga) <= ctol * sqrt(al) * sqrt(be)) continue;
                if (lane == 0) rotated = 1;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double s = c * t;
                for (int r = lane; r < p; r += 32) {
                    const double x = wa[r], y = wb[r];
                    wa[r] = c * x - s * y;
                    wb[r] = s * x + c * y;
                }
                double *va = V + (int64_t)a * p, *vb = V + (int64_t)b * p;
                for (int r = lane; r < p; r += 32) {
                    const double x = va[r], y = vb[r];
                    va[r] = c * x - s * y;
                    vb[r] = s * x + c * y;
                }
            }
            __syncthreads();
        }
        const int any = rotated;
        __syncthreads();
        if (!any) {
            conv = true;
            break;
        }
    }
    if (threadIdx.x == 0) {
        ctrl->svd_sweeps = sweep;
        ctrl->svd_status = conv ? 0 : (int)SVDSC_ESVD_NOCONV;
    }
}

// rotation parameters from t = tan(theta), pinned rounding (no contraction) so
// that the W kernel and the V (log-apply) kernel produce bitwise equal c, s
__device__ __forceinline__ void rot_cs(double t, double &c, double &s) {
    c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
    s = __dmul_rn(c, t);
}

// One-sided Jacobi with W = T(1:p,1:p) resident in the shared memory of a
// thread-block cluster (C CTAs own ceil(p/C) columns each; pairs whose columns
// live in another CTA are reached through distributed shared memory).  The
// tangent of every rotation is logged (0 = no rotation) so that V = J_1 J_2 ...
// can be formed afterwards by k_apply_log, row-parallel, off the critical path.
__global__ void __launch_bounds__(1024) k_jacobi_cluster(int p, int ncc, const double *__restrict__ W0, double *Wout,
                                                         double *tlog, int max_sweeps, Ctrl *ctrl, const int *abort,
                                                         double ctol) {
    if (aborted(abort)) return;
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), me = (int)cl.block_rank();
    extern __shared__ double Wl[];
    __shared__ int rot_flag[2];  // by sweep parity: the flag of sweep s+1 is cleared during sweep s
    const double tiny = *(volatile double *)&ctrl->svd_tiny;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int c0 = me * ncc;
    for (int idx = threadIdx.x; idx < ncc * p; idx += blockDim.x) {
        const int col = c0 + idx / p, r = idx % p;
        Wl[idx] = (col < p) ? W0[r + (int64_t)col * p] : 0.0;
    }
    if (threadIdx.x == 0) rot_flag[0] = rot_flag[1] = 0;
    cl.sync();
    const int pe = p + (p & 1), npairs = pe / 2;
    int sweep;
    bool conv = false;
    for (sweep = 1; sweep <= max_sweeps; sweep++) {
        int *flag = &rot_flag[sweep & 1];
        for (int rnd = 0; rnd < pe - 1; rnd++) {
            double *logr = tlog + ((int64_t)(sweep - 1) * (pe - 1) + rnd) * npairs;
            for (int q = me * nw + wid; q < npairs; q += C * nw) {
                int a, b;
                rr_pair(pe, rnd, q, a, b);
                double t = 0.0;
                if (b < p) {
                    const int oa = a / ncc, ob = b / ncc;
                    double *wa = Wl + (a - oa * ncc) * p, *wb = Wl + (b - ob * ncc) * p;
                    if (oa != me) wa = cl.map_shared_rank(wa, oa);
                    if (ob != me) wb = cl.map_shared_rank(wb, ob);
                    double al = 0.0, be = 0.0, ga = 0.0;
                    for (int r = lane; r < p; r += 32) {
                        const double x = wa[r], y = wb[r];
                        al = fma(x, x, al);
                        be = fma(y, y, be);
                        ga = fma(x, y, ga);
                    }
                    al = warp_sum(al);
                    be = warp_sum(be);
                    ga = warp_sum(ga);
                    if (sqrt(al) > tiny && sqrt(be) > tiny && fabs(ga) > ctol * sqrt(al) * sqrt(be)) {
                        const double zeta = (be - al) / (2.0 * ga);
                        t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                        double c, s;
                        rot_cs(t, c, s);
                        for (int r = lane; r < p; r += 32) {
                            const double x = wa[r], y = wb[r];
                            wa[r] = c * x - s * y;
                            wb[r] = s * x + c * y;
                        }
                        if (lane == 0) *flag = 1;
                    }
                }
                if (lane == 0) logr[q] = t;
            }
            cl.sync();
            // every CTA has read the previous sweep's flags by now: recycle that slot
            if (rnd == 0 && threadIdx.x == 0) rot_flag[(sweep + 1) & 1] = 0;
        }
        int any = 0;
        for (int r = 0; r < C; r++) any |= *cl.map_shared_rank(flag, r);
        if (!any) {
            conv = true;
            break;
        }
    }
    for (int idx = threadIdx.x; idx < ncc * p; idx += blockDim.x) {
        const int col = c0 + idx / p, r = idx % p;
        if (col < p) Wout[r + (int64_t)col * p] = Wl[idx];
    }
    if (me == 0 && threadIdx.x == 0) {
        ctrl->svd_sweeps = conv ? sweep : max_sweeps;
        ctrl->svd_status = conv ? 0 : (int)SVDSC_ESVD_NOCONV;
    }
    cl.sync();
}

// V = J_1 J_2 ... (the logged rotations) for R rows of V per CTA: each row of V
// evolves independently (row r of V = e_r^T J_1 J_2 ...).  The log is staged
// through shared memory in chunks of KR rounds with cp.async double buffering.
constexpr int kLogRounds = 16;
__global__ void k_apply_log(int p, const double *__restrict__ tlog, const Ctrl *ctrl, double *V, int R,
                            const int *abort) {
    if (aborted(abort)) return;
    extern __shared__ double sm[];
    const int pe = p + (p & 1), npairs = pe / 2;
    const int nsweeps = ctrl->svd_sweeps;
    const int64_t total_rounds = (int64_t)nsweeps * (pe - 1);
    double *rows = sm;                           // R x p
    double *buf = rows + (int64_t)R * p;         // 2 x kLogRounds x npairs
    const int chunk = kLogRounds * npairs;
    const int r0 = blockIdx.x * R;
    for (int idx = threadIdx.x; idx < R * p; idx += blockDim.x) {
        const int i = idx / p, j = idx % p;
        rows[idx] = (r0 + i == j) ? 1.0 : 0.0;
    }
    auto load_chunk = [&](int64_t first_round, double *dst) {
        const int64_t nrem = total_rounds - first_round;
        const int n = (int)min((int64_t)kLogRounds, max((int64_t)0, nrem)) * npairs;
        const double *src = tlog + first_round * npairs;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst + i);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr), "l"(src + i));
        }
        asm volatile("cp.async.commit_group;");
    };
    if (total_rounds > 0) load_chunk(0, buf);
    int cur = 0;
    for (int64_t base = 0; base < total_rounds; base += kLogRounds) {
        if (base + kLogRounds < total_rounds) {
            load_chunk(base + kLogRounds, buf + (cur ^ 1) * chunk);
            asm volatile("cp.async.wait_group 1;");
        } else {
            asm volatile("cp.async.wait_group 0;");
        }
        __syncthreads();
        const double *lg = buf + cur * chunk;
        const int nr = (int)min((int64_t)kLogRounds, total_rounds - base);
        for (int k = 0; k < nr; k++) {
            const int rnd = (int)((base + k) % (pe - 1));
            const int q = threadIdx.x;
            if (q < npairs) {
                int a, b;
                rr_pair(pe, rnd, q, a, b);
                const double t = lg[k * npairs + q];
                if (b < p && t != 0.0) {
                    double c, s;
                    rot_cs(t, c, s);
                    for (int i = 0; i < R; i++) {
                        double *row = rows + i * p;
                        const double x = row[a], y = row[b];
                        row[a] = c * x - s * y;
                        row[b] = s * x + c * y;
                    }
                }
            }
            __syncthreads();
        }
        cur ^= 1;
    }
    for (int idx = threadIdx.x; idx < R * p; idx += blockDim.x) {
        const int i = idx / p, j = idx % p;
        if (r0 + i < p) V[(r0 + i) + (int64_t)j * p] = rows[idx];
    }
}

// norms, descending sort (ties: natural order), U = W / sigma, zero-sigma
// completion of the first kneed columns, sign rule.
__global__ void __launch_bounds__(1024) k_svd_finish(int p, const double *__restrict__ W, const double *__restrict__ V,
                                                     double *Uh, double *Sh, double *Vh, int kneed, const Ctrl *ctrl,
                                                     const int *abort) {
    if (aborted(abort)) return;
    const double tiny = ctrl->svd_tiny;
    __shared__ double sig[kMaxP];
    __shared__ int dest[kMaxP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = wid; j < p; j += nw) {
        double s = 0.0;
        for (int r = lane; r < p; r += 32) {
            const double x = W[r + (int64_t)j * p];
            s = fma(x, x, s);
        }
        s = warp_sum(s);
        if (lane == 0) sig[j] = (sqrt(s) > tiny) ? sqrt(s) : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < p; j += blockDim.x) {
        int rk = 0;
        const double sj = sig[j];
        for (int l = 0; l < p; l++) rk += (sig[l] > sj) || (sig[l] == sj && l < j);
        dest[j] = rk;
    }
    __syncthreads();
    for (int j = wid; j < p; j += nw) {
        const int d = dest[j];
        const double sj = sig[j];
        if (lane == 0) Sh[d] = sj;
        for (int r = lane; r < p; r += 32) {
            Vh[r + (int64_t)d * p] = V[r + (int64_t)j * p];
            Uh[r + (int64_t)d * p] = sj > 0.0 ? W[r + (int64_t)j * p] / sj : 0.0;
        }
    }
    __syncthreads();
    // zero singular values among the first kneed: complete U with the standard
    // basis vector whose residual after two Gram-Schmidt passes against the
    // previous columns is largest (the oracle's rule).  Rare: exact rank loss.
    if (wid == 0) {
        for (int d = 0; d < kneed && d < p; d++) {
            if (Sh[d] > 0.0) continue;
            double *ud = Uh + (int64_t)d * p;
            int best = 0;
            double bestn = -1.0;
            for (int pick = 0; pick < 2; pick++) {
                const int e0 = pick ? best : 0, e1 = pick ? best + 1 : p;
                for (int e = e0; e < e1; e++) {
                    for (int r = lane; r < p; r += 32) ud[r] = (r == e) ? 1.0 : 0.0;
                    __syncwarp();
                    for (int pass = 0; pass < 2; pass++)
                        for (int jj = 0; jj < d; jj++) {
                            const double *uj = Uh + (int64_t)jj * p;
                            double dd = 0.0;
                            for (int r = lane; r < p; r += 32) dd = fma(uj[r], ud[r], dd);
                            dd = warp_sum(dd);
                            for (int r = lane; r < p; r += 32) ud[r] -= dd * uj[r];
                            __syncwarp();
                        }
                    double nn = 0.0;
                    for (int r = lane; r < p; r += 32) nn = fma(ud[r], ud[r], nn);
                    nn = sqrt(warp_sum(nn));
                    if (!pick && nn > bestn) {
                        bestn = nn;
                        best = e;
                    }
                    if (pick)
                        for (int r = lane; r < p; r += 32) ud[r] /= nn;
                    __syncwarp();
                }
            }
        }
    }
    __syncthreads();
    // sign rule: the largest-|.| entry of u_j (first index on ties) made >= 0
    for (int j = wid; j < p; j += nw) {
        double *uj = Uh + (int64_t)j * p;
        double best = -1.0;
        int bi = p;
        for (int r = lane; r < p; r += 32) {
            const double a = fabs(uj[r]);
            if (a > best) {
                best = a;
                bi = r;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        const bool flip = uj[bi] < 0.0;
        if (flip) {
            double *vj = Vh + (int64_t)j * p;
            for (int r = lane; r < p; r += 32) {
                uj[r] = -uj[r];
                vj[r] = -vj[r];
            }
        }
    }
}

__global__ void k_residuals(int t, int k, const double *__restrict__ T, int ldt, const double *__restrict__ Uh,
                            const double *__restrict__ Sh, double tol, double *resid, Ctrl *ctrl, const int *abort) {
    if (aborted(abort)) return;
    __shared__ int nconv, rankdef;
    __shared__ double mx[32];
    if (threadIdx.x == 0) {
        nconv = 1;
        rankdef = 0;
    }
    __syncthreads();
    const double beta_t = T[(t - 1) + (int64_t)t * ldt];
    double m = 0.0;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const double num = fabs(beta_t * Uh[(t - 1) + (int64_t)j * t]);
        double r;
        if (Sh[j] > 0.0) r = num / Sh[j];
        else if (num <= 1e-14) r = 0.0;
        else {
            r = num;
            rankdef = 1;
        }
        if (resid) resid[j] = r;
        if (!(r < tol)) nconv = 0;  // strict '<'
        m = fmax(m, r);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) mx[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) mm = fmax(mm, mx[i]);
        ctrl->max_resid = mm;
        ctrl->converged = nconv;
        ctrl->rankdef = rankdef;
    }
}

__global__ void k_restart_T(int t, int k, double *T, int ldt, const double *__restrict__ Uh,
                            const double *__restrict__ Sh, double *rho) {
    const double beta_t = T[(t - 1) + (int64_t)t * ldt];
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) rho[j] = beta_t * Uh[(t - 1) + (int64_t)j * t];
    const int n = (t + 1) * ldt;
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) T[idx] = 0.0;
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        T[j + (int64_t)j * ldt] = Sh[j];
        T[j + (int64_t)k * ldt] = rho[j];
    }
}

// Qout(:, 0:k) = Q(:, 0:t) W(:, 0:k) for a row tile of RT rows staged in shared
// memory (in place safe: a tile is fully read before any of its rows is written).
__global__ void __launch_bounds__(256) k_recombine(int64_t N, int t, int k, const double *Q, int64_t ldq,
                                                   const double *__restrict__ Wm, int ldw, double *Qout,
                                                   int64_t ldo, int RT) {
    extern __shared__ double tile[];  // t x (RT+1)
    const int LDT = RT + 1;
    const int64_t ntiles = (N + RT - 1) / RT;
    for (int64_t tI = blockIdx.x; tI < ntiles; tI += gridDim.x) {
        const int64_t r0 = tI * RT;
        const int nr = (int)min((int64_t)RT, N - r0);
        for (int idx = threadIdx.x; idx < t * RT; idx += blockDim.x) {
            const int j = idx / RT, q = idx - j * RT;
            tile[j * LDT + q] = (q < nr) ? Q[r0 + q + (int64_t)j * ldq] : 0.0;
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < k * RT; idx += blockDim.x) {
            const int j = idx / RT, q = idx - j * RT;
            const double *wj = Wm + (int64_t)j * ldw;
            double s = 0.0;
            for (int l = 0; l < t; l++) s = fma(tile[l * LDT + q], __ldg(wj + l), s);
            if (q < nr) Qout[r0 + q + (int64_t)j * ldo] = s;
        }
        __syncthreads();
    }
}

}  // namespace

size_t small_svd_log_doubles(int p) {
    const int64_t pe = p + (p & 1);
    return (size_t)(50 * (pe - 1) * (pe / 2));
}

void small_svd(int p, const double *Tsrc, int ldt, double *W, double *Vw, double *Uh, double *Sh, double *Vh,
               int kneed, Ctrl *ctrl, const int *abort, double *tlog, cudaStream_t s) {
    k_copy_T<<<1, 1024, 0, s>>>(p, Tsrc, ldt, W, Vw, ctrl, abort);
    count_launch();
    const double ctol = 2.0 * (double)p * 2.220446049250313e-16;  // reading Q10a
    bool done = false;
    if (tlog) {
        // smallest cluster whose shared memory holds W
        int C = 1;
        while (C <= 16 && (size_t)((p + C - 1) / C) * p * 8 > 200 * 1024) C <<= 1;
        if (C <= 16) {
            const int ncc = (p + C - 1) / C;
            const size_t smem = (size_t)ncc * p * 8;
            cudaFuncSetAttribute(k_jacobi_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
            if (C > 8) cudaFuncSetAttribute(k_jacobi_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(1024);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = C;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaLaunchKernelEx(&cfg, k_jacobi_cluster, p, ncc, (const double *)W, W, tlog, 50, ctrl, abort, ctol) ==
                cudaSuccess) {
                count_launch();
                const int pe = p + (p & 1), npairs = pe / 2;
                const int R = 4;
                const int threads = std::max(32, ((npairs + 31) / 32) * 32);
                const size_t smem2 = ((size_t)R * p + 2 * (size_t)kLogRounds * npairs) * 8;
                cudaFuncSetAttribute(k_apply_log, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                k_apply_log<<<(p + R - 1) / R, threads, smem2, s>>>(p, tlog, ctrl, Vw, R, abort);
                count_launch();
                done = true;
            } else {
                cudaGetLastError();  // clear and fall back
            }
        }
    }
    if (!done) {
        k_jacobi<<<1, 1024, 0, s>>>(p, W, Vw, ctrl, abort, ctol, 50);
        count_launch();
    }
    k_svd_finish<<<1, 1024, 0, s>>>(p, W, Vw, Uh, Sh, Vh, kneed, ctrl, abort);
    count_launch();
}

void residuals(int t, int k, const double *T, int ldt, const double *Uh, const double *Sh, double tol,
               double *resid, Ctrl *ctrl, const int *abort, cudaStream_t s) {
    k_residuals<<<1, 256, 0, s>>>(t, k, T, ldt, Uh, Sh, tol, resid, ctrl, abort);
    count_launch();
}

void restart_T(int t, int k, double *T, int ldt, const double *Uh, const double *Sh, double *rho, cudaStream_t s) {
    k_restart_T<<<1, 1024, 0, s>>>(t, k, T, ldt, Uh, Sh, rho);
    count_launch();
}

void recombine(int64_t N, int t, int k, const double *Q, int64_t ldq, const double *W, int ldw, double *Qout,
               int64_t ldo, int nsm, cudaStream_t s) {
    int RT = 64;
    while (RT > 8 && (size_t)t * (RT + 1) * 8 > 100 * 1024) RT >>= 1;
    const size_t smem = (size_t)t * (RT + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_recombine, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const int64_t ntiles = (N + RT - 1) / RT;
    const int nb = (int)std::min<int64_t>(ntiles, (int64_t)nsm * 2);
    k_recombine<<<std::max(nb, 1), 256, smem, s>>>(N, t, k, Q, ldq, W, ldw, Qout, ldo, RT);
    count_launch();
}

void copy_col(int64_t N, const double *src, double *dst, cudaStream_t s) {
    cudaMemcpyAsync(dst, src, N * sizeof(double), cudaMemcpyDeviceToDevice, s);
}

void fill_zero(double *p, int64_t n, cudaStream_t s) { cudaMemsetAsync(p, 0, n * sizeof(double), s); }

}  // namespace svdsc
