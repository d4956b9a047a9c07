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
#include <cstdio>
#include <cstdlib>

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

__device__ __forceinline__ double rcp_approx(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_approx(double x) {
    double y;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

// rotation parameters from t = tan(theta): c = (1 + t^2)^(-1/2) to ~1 ulp
// (hardware rsqrt approximation + two Newton steps), s = c t.  Pinned
// rounding (explicit _rn intrinsics, no contraction choices left to the
// compiler) so that the W kernel and the V (log-apply) kernel produce bitwise
// equal c, s from the logged t.
__device__ __forceinline__ void rot_cs(double t, double &c, double &s) {
    const double x = __fma_rn(t, t, 1.0);
    const double hx = __dmul_rn(0.5, x);
    double y = rsqrt_approx(x);
    y = __dmul_rn(y, __fma_rn(-hx, __dmul_rn(y, y), 1.5));
    y = __dmul_rn(y, __fma_rn(-hx, __dmul_rn(y, y), 1.5));
    c = y;
    s = __dmul_rn(c, t);
}

// tangent of the Jacobi angle for the pair (alpha, beta, gamma): only the
// convergence rate depends on its accuracy (the rotation built from it by
// rot_cs is orthogonal to working precision), so fast approximate reciprocal /
// rsqrt are used: zeta = (beta - alpha) / (2 gamma), t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)).
__device__ __forceinline__ double jacobi_tan(double al, double be, double gam) {
    const double zeta = (be - al) * 0.5 * rcp_approx(gam);
    const double az = fabs(zeta);
    double t;
    if (az > 1e100) {
        t = 0.5 * rcp_approx(az);
    } else {
        const double r = fma(az, az, 1.0);
        t = rcp_approx(az + r * rsqrt_approx(r));
    }
    return zeta >= 0.0 ? t : -t;
}

// ---------------------------------------------------------------------------
// Block one-sided Jacobi on a thread-block cluster (B200: up to 16 CTAs,
// distributed shared memory).  The pe = p + (p odd) columns are cut into 2C
// half-blocks of h columns; CTA c holds two half-blocks in its shared memory.
// Block round 0 of a sweep runs a full local round-robin sweep over the CTA's
// 2h columns (all pairs, LDS only, __syncthreads between local rounds); every
// later block round runs only the h cross rounds between its two half-blocks,
// with the slot-0 column of each warp held in registers (every pair still
// meets once per sweep; 40% fewer rounds than a full local sweep per block
// round, and half the shared-memory traffic per rotation).  Between
// block rounds the half-blocks move along the circle-method tournament (one
// DSMEM pull into registers, cluster barrier, store), so every pair of
// half-blocks meets once per block sweep.  Every rotation is logged as
// (t = tan theta, a, b) for k_apply_log; rotations of one local round (all
// CTAs) touch disjoint columns, so replaying them round by round is exact.
struct RotLog {
    double c, s;      // the rotation as applied to W (c = s = 0: no rotation)
    int32_t a, b;     // global column pair, a < b
    int64_t pad;      // 32-byte entries: 16-byte cp.async staging
};

// circle-method tournament over 2C players (player 0 fixed, m = 2C - 1)
__device__ __forceinline__ int hb_at(int C, int r, int c, int slot) {
    const int m = 2 * C - 1;
    if (slot == 0) return c == 0 ? 0 : ((c - 1 - r) % m + m) % m + 1;
    return ((m - 1 - c - r) % m + m) % m + 1;
}
// where (cta, slot) is player P in round r
__device__ __forceinline__ void hb_loc(int C, int r, int P, int &cta, int &slot) {
    if (P == 0) {
        cta = 0;
        slot = 0;
        return;
    }
    const int m = 2 * C - 1;
    const int k = (P - 1 + r) % m;
    if (k < C - 1) {
        cta = k + 1;
        slot = 0;
    } else {
        cta = m - 1 - k;
        slot = 1;
    }
}

// rounds of one sweep: block round 0 = full local round robin over 2h columns
// (2h - 1 rounds), each later block round = the h cross rounds of its two
// half-blocks; (2C - 1) block rounds
__host__ __device__ __forceinline__ int64_t jacobi_rounds_per_sweep(int C, int h) {
    return (int64_t)(2 * h - 1) + (int64_t)(2 * C - 2) * h;
}

// alpha = |a|^2, beta = |b|^2, gamma = a.b over the warp's rows (two
// interleaved FMA chains per sum, xor-butterfly over the 32 lanes)
template <int kRPL>
__device__ __forceinline__ void pair_sums(const double (&a)[kRPL], const double (&b)[kRPL], double &al, double &be,
                                          double &gam) {
    double al1 = 0.0, be1 = 0.0, ga1 = 0.0;
    al = be = gam = 0.0;
#pragma unroll
    for (int u = 0; u < kRPL; u += 2) {
        al = fma(a[u], a[u], al);
        be = fma(b[u], b[u], be);
        gam = fma(a[u], b[u], gam);
        if (u + 1 < kRPL) {
            al1 = fma(a[u + 1], a[u + 1], al1);
            be1 = fma(b[u + 1], b[u + 1], be1);
            ga1 = fma(a[u + 1], b[u + 1], ga1);
        }
    }
    al += al1;
    be += be1;
    gam += ga1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, off);
        be += __shfl_xor_sync(0xffffffffu, be, off);
        gam += __shfl_xor_sync(0xffffffffu, gam, off);
    }
}

constexpr int kExR = 20;  // registers per thread per slot for the half-block exchange (h*p <= 20*640)

constexpr int kMaxRPL = 20;   // rows per lane held in registers: p <= 32 * kMaxRPL
constexpr int kJThreads = 640; // 20 warps: one warp per pair, <= 20 pairs per CTA
constexpr int kJMaxH = 12;     // preferred half-block width (measured, tools/time_ops.py)
constexpr int kMaxPairs = kJThreads / 32;

template <bool CL, int kRPL>
__global__ void __launch_bounds__(kJThreads) k_jacobi_block(int p, int h, const double *__restrict__ W0, double *Wout,
                                                       RotLog *rlog, int max_sweeps, Ctrl *ctrl, const int *abort,
                                                       double ctol, int use_bulk) {
    if (aborted(abort)) return;
    cg::cluster_group cl = cg::this_cluster();
    const int C = CL ? (int)cl.num_blocks() : 1;
    const int me = CL ? (int)cl.block_rank() : 0;
    extern __shared__ __align__(16) double Wsm[];  // slot s, local column i: Wl + (s*h + i)*p
    // bulk-copy exchange: two half-block buffer sets, Wl = the current one
    // (push model: every CTA sends its two half-blocks to their next owners
    // with cp.async.bulk shared::cta -> shared::cluster, completing on the
    // receiver's mbarrier); else one set and a register pull through DSMEM
    const bool bulk = CL && use_bulk;
    double *Wl = Wsm;
    __shared__ __align__(8) uint64_t xbar;
    __shared__ int rot_flag[2];
    __shared__ int src_cta[2], src_slot[2];
    const double tiny = *(volatile double *)&ctrl->svd_tiny;
    const double tiny2 = tiny * tiny;
    const double ctol2 = ctol * ctol;
    constexpr int kG = 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gl = lane;
    const int ngrp = blockDim.x / kG;
    const int m = 2 * C - 1;
    const int H2 = 2 * h;
    __shared__ unsigned short pair_tab[2 * kMaxPairs * 2 * kMaxPairs];  // [lr][q] = i | j << 8
    __shared__ int gcol[2 * kMaxPairs];                                  // local column -> global
    int hb[2] = {hb_at(C, 0, me, 0), hb_at(C, 0, me, 1)};
    for (int idx = threadIdx.x; idx < (H2 - 1) * h; idx += blockDim.x) {
        int i, j;
        rr_pair(H2, idx / h, idx % h, i, j);
        pair_tab[idx] = (unsigned short)(i | (j << 8));
    }
    for (int lc = threadIdx.x; lc < H2; lc += blockDim.x) gcol[lc] = hb[lc / h] * h + (lc % h);
    for (int idx = threadIdx.x; idx < H2 * p; idx += blockDim.x) {
        const int lc = idx / p, r = idx % p;
        const int col = hb[lc / h] * h + (lc % h);
        Wl[idx] = (col < p) ? W0[r + (int64_t)col * p] : 0.0;
    }
    if (threadIdx.x == 0) {
        rot_flag[0] = rot_flag[1] = 0;
        if (bulk) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&xbar))
                         : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    }
    unsigned xphase = 0;
    if (CL) cl.sync(); else __syncthreads();
    const int64_t per_round = (int64_t)C * h;
    const int lrounds = H2 - 1;
    const int64_t rps = jacobi_rounds_per_sweep(C, h);
    int sweep;
    bool conv = false;
    for (sweep = 1; sweep <= max_sweeps; sweep++) {
        int *flag = &rot_flag[sweep & 1];
        for (int br = 0; br < m; br++) {
            if (br == 0) {
            // block round 0: all pairs of the CTA's 2h columns (local round robin, shared memory)
            for (int lr = 0; lr < lrounds; lr++) {
                RotLog *logr = rlog + ((int64_t)(sweep - 1) * rps + lr) * per_round + (int64_t)me * h;
                for (int qb = wid * (32 / kG); qb < h; qb += ngrp) {
                    const int q = qb + lane / kG;
                    int i = 0, j = 0;
                    if (q < h) {
                        const unsigned pr = pair_tab[lr * h + q];
                        i = pr & 0xff;
                        j = pr >> 8;
                    }
                    const int ga = gcol[i], gb = gcol[j];
                    const bool live = (q < h) && ga < p && gb < p;
                    // the pair's columns, oriented (lower global index, higher) as in the oracle
                    double *pa = Wl + (int64_t)(ga < gb ? i : j) * p, *pb = Wl + (int64_t)(ga < gb ? j : i) * p;
                    double xr[kRPL], yr[kRPL];
#pragma unroll
                    for (int u = 0; u < kRPL; u++) {
                        const int r = gl + kG * u;
                        const bool ok = live && r < p;
                        xr[u] = ok ? pa[r] : 0.0;
                        yr[u] = ok ? pb[r] : 0.0;
                    }
                    double al, be, gam;
                    pair_sums<kRPL>(xr, yr, al, be, gam);
                    double c = 0.0, s = 0.0;
                    if (live && al > tiny2 && be > tiny2 && gam * gam > ctol2 * (al * be)) {
                        rot_cs(jacobi_tan(al, be, gam), c, s);
#pragma unroll
                        for (int u = 0; u < kRPL; u++) {
                            const int r = gl + kG * u;
                            if (r < p) {
                                pa[r] = c * xr[u] - s * yr[u];
                                pb[r] = s * xr[u] + c * yr[u];
                            }
                        }
                        if (gl == 0) *flag = 1;
                    }
                    if (gl == 0 && q < h) {
                        RotLog e;
                        e.c = c;
                        e.s = s;
                        e.a = min(ga, gb);
                        e.b = max(ga, gb);
                        logr[q] = e;
                    }
                }
                __syncthreads();
            }
            } else {
            // block rounds >= 1: only the h^2 cross pairs of the two half-blocks
            // (pairs inside a half-block were rotated in block round 0).  Warp i
            // keeps column X[i] (slot 0) in registers for the whole block round
            // and meets Y[(i + r) mod h] (slot 1) in round r: one column read and
            // written per rotation instead of two.
            const bool has = wid < h;
            const int gx = has ? gcol[wid] : p;
            double xr[kRPL];
#pragma unroll
            for (int u = 0; u < kRPL; u++) {
                const int r = gl + kG * u;
                xr[u] = (has && r < p) ? Wl[(int64_t)wid * p + r] : 0.0;
            }
            const int64_t rbase = (int64_t)(sweep - 1) * rps + lrounds + (int64_t)(br - 1) * h;
            int jy = wid < h ? wid : 0;  // (wid + rr) mod h, advanced without a division
            for (int rr = 0; rr < h; rr++, jy = (jy + 1 == h) ? 0 : jy + 1) {
                if (has) {
                    const int j = h + jy;
                    const int gy = gcol[j];
                    const bool live = gx < p && gy < p;
                    double *py = Wl + (int64_t)j * p;
                    double yr[kRPL];
#pragma unroll
                    for (int u = 0; u < kRPL; u++) {
                        const int r = gl + kG * u;
                        yr[u] = (live && r < p) ? py[r] : 0.0;
                    }
                    const bool xlow = gx < gy;
                    double al, be, gam;
                    if (xlow) pair_sums<kRPL>(xr, yr, al, be, gam);
                    else pair_sums<kRPL>(yr, xr, al, be, gam);
                    double c = 0.0, s = 0.0;
                    if (live && al > tiny2 && be > tiny2 && gam * gam > ctol2 * (al * be)) {
                        rot_cs(jacobi_tan(al, be, gam), c, s);
                        // (A, B) = (lower, higher): A' = c A - s B, B' = s A + c B; with
                        // X the higher column this is X' = c X + s Y, Y' = c Y - s X,
                        // i.e. the same form with s -> -s
                        const double sx = xlow ? s : -s;
#pragma unroll
                        for (int u = 0; u < kRPL; u++) {
                            const double x = xr[u], y = yr[u];
                            xr[u] = c * x - sx * y;
                            yr[u] = sx * x + c * y;
                            const int r = gl + kG * u;
                            if (r < p) py[r] = yr[u];
                        }
                        if (gl == 0) *flag = 1;
                    }
                    if (gl == 0) {
                        RotLog e;
                        e.c = c;
                        e.s = s;
                        e.a = min(gx, gy);
                        e.b = max(gx, gy);
                        rlog[(rbase + rr) * per_round + (int64_t)me * h + wid] = e;
                    }
                }
                __syncthreads();
            }
            if (has) {
#pragma unroll
                for (int u = 0; u < kRPL; u++) {
                    const int r = gl + kG * u;
                    if (r < p) Wl[(int64_t)wid * p + r] = xr[u];
                }
            }
            __syncthreads();
            }
            if (CL && m > 1 && bulk) {
                const int rn = (br + 1) % m;
                const int n = h * p;
                double *Wn = (Wl == Wsm) ? Wsm + 2 * n : Wsm;  // the other buffer set
                const unsigned bar = (unsigned)__cvta_generic_to_shared(&xbar);
                // every thread's generic-proxy writes of its half-block columns are
                // ordered before the async-proxy (bulk copy) reads that follow
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (threadIdx.x == 0) {
                    // two incoming half-blocks; armed before the cluster barrier
                    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                                 "r"((unsigned)(2 * n * 8))
                                 : "memory");
                }
                cl.sync();  // block round done everywhere; every CTA's barrier is armed
                if (threadIdx.x < 2) {
                    const int sl = threadIdx.x;
                    int ct, ds;
                    hb_loc(C, rn, hb_at(C, br, me, sl), ct, ds);  // where my slot-sl half-block goes
                    const unsigned src = (unsigned)__cvta_generic_to_shared(Wl + (int64_t)sl * n);
                    const unsigned dloc = (unsigned)__cvta_generic_to_shared(Wn + (int64_t)ds * n);
                    unsigned dst, rbar;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(dloc), "r"(ct));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar), "r"(ct));
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            dst),
                        "r"(src), "r"((unsigned)(n * 8)), "r"(rbar)
                        : "memory");
                }
                // wait for my two incoming half-blocks
                asm volatile(
                    "{\n.reg .pred P1;\nXW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra XW_%=;\n}\n" ::"r"(
                        bar),
                    "r"(xphase)
                    : "memory");
                xphase ^= 1;
                Wl = Wn;
                hb[0] = hb_at(C, rn, me, 0);
                hb[1] = hb_at(C, rn, me, 1);
                for (int lc = threadIdx.x; lc < H2; lc += blockDim.x) gcol[lc] = hb[lc / h] * h + (lc % h);
                __syncthreads();
            } else if (CL && m > 1) {
                // move to round br+1 (after the last block round the circle is back at round 0)
                const int rn = (br + 1) % m;
                if (threadIdx.x < 2) {
                    int ct, sl;
                    hb_loc(C, br, hb_at(C, rn, me, threadIdx.x), ct, sl);
                    src_cta[threadIdx.x] = ct;
                    src_slot[threadIdx.x] = sl;
                }
                cl.sync();  // local sweeps done everywhere; sources known
                double reg[2][kExR];
                const int n = h * p;
#pragma unroll
                for (int sl = 0; sl < 2; sl++) {
                    const double *src = Wl + (int64_t)src_slot[sl] * n;
                    if (src_cta[sl] != me) src = cl.map_shared_rank(src, src_cta[sl]);
#pragma unroll
                    for (int u = 0; u < kExR; u++) {
                        const int idx = threadIdx.x + u * blockDim.x;
                        reg[sl][u] = (idx < n) ? src[idx] : 0.0;
                    }
                }
                cl.sync();  // every CTA has pulled its new half-blocks
#pragma unroll
                for (int sl = 0; sl < 2; sl++)
#pragma unroll
                    for (int u = 0; u < kExR; u++) {
                        const int idx = threadIdx.x + u * blockDim.x;
                        if (idx < n) Wl[(int64_t)sl * n + idx] = reg[sl][u];
                    }
                hb[0] = hb_at(C, rn, me, 0);
                hb[1] = hb_at(C, rn, me, 1);
                for (int lc = threadIdx.x; lc < H2; lc += blockDim.x) gcol[lc] = hb[lc / h] * h + (lc % h);
                __syncthreads();
            }
        }
        // the next sweep's flag is cleared before the barrier: after it, other
        // warps may already be setting it in the next sweep
        if (threadIdx.x == 0) rot_flag[(sweep + 1) & 1] = 0;
        if (CL) cl.sync(); else __syncthreads();
        int any = 0;
        if (CL) {
            for (int r = 0; r < C; r++) any |= *cl.map_shared_rank(flag, r);
        } else {
            any = *flag;
        }
        if (CL) cl.sync(); else __syncthreads();
        if (!any) {
            conv = true;
            break;
        }
    }
    for (int idx = threadIdx.x; idx < H2 * p; idx += blockDim.x) {
        const int lc = idx / p, r = idx % p;
        const int col = hb[lc / h] * h + (lc % h);
        if (col < p) Wout[r + (int64_t)col * p] = Wl[idx];
    }
    if (me == 0 && threadIdx.x == 0) {
        ctrl->svd_sweeps = conv ? sweep : max_sweeps;
        ctrl->svd_status = conv ? 0 : (int)SVDSC_ESVD_NOCONV;
    }
    if (CL) cl.sync();
}

// ---------------------------------------------------------------------------
// Register Jacobi for p <= 64 (pe / 2 <= 32 pair slots, one CTA).  Pair slot q
// is a group of kJG = 8 lanes holding the slot's two columns of W AND of V in
// registers (lane g: rows g + 8 u, u < RL), so V is accumulated as the
// rotations are applied (no rotation log, no replay launch) and T is read in
// place.  8-lane groups keep the per-round reductions to 3 butterfly levels
// and 4 pairs per warp (one warp per pair spent most of a round in shuffles).
// Circle method with position 0 fixed: in round r position i >= 1 holds
// column ((i - 1 - r) mod (pe - 1)) + 1 and slot q pairs positions q and
// pe - 1 - q; between rounds every column moves one position through a
// double-buffered shared-memory exchange (one barrier per round; position
// stride = 8 mod 16 doubles so the 4 groups of a warp hit both bank halves).
// After pe - 1 rounds (one sweep) every pair has met once and the columns are
// back in place.  Rotation rule, threshold and orientation (lower global
// column first) as in k_jacobi_block; ctrl->svd_tiny = p eps ||T||_F as in
// k_copy_T.
constexpr int kJG = 8;

template <int RL>
__device__ __forceinline__ void group_pair_sums(const double (&a)[RL], const double (&b)[RL], double &al, double &be,
                                                double &gam) {
    al = be = gam = 0.0;
#pragma unroll
    for (int u = 0; u < RL; u++) {
        al = fma(a[u], a[u], al);
        be = fma(b[u], b[u], be);
        gam = fma(a[u], b[u], gam);
    }
#pragma unroll
    for (int off = kJG / 2; off > 0; off >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, off);
        be += __shfl_xor_sync(0xffffffffu, be, off);
        gam += __shfl_xor_sync(0xffffffffu, gam, off);
    }
}

template <int RL>
__global__ void __launch_bounds__(256) k_jacobi_reg(int p, const double *__restrict__ T, int ldt, double *Wout,
                                                    double *Vout, Ctrl *ctrl, const int *abort, double ctol,
                                                    int max_sweeps) {
    if (aborted(abort)) return;
    constexpr int R = kJG * RL;     // rows per column (p <= R)
    constexpr int PS = 2 * R + 8;   // position stride: W column, V column, pad
    extern __shared__ __align__(16) double xs[];  // [2 buffers][pe positions][PS]
    __shared__ double red[32];
    const int pe = p + (p & 1), np2 = pe / 2, m = pe - 1;
    const int g = threadIdx.x % kJG, q = threadIdx.x / kJG;
    const bool slot = q < np2;  // lanes past the last slot hold zero columns
    const int ct0 = slot ? q : pe, cb0 = slot ? pe - 1 - q : pe;  // columns at round 0
    double wt[RL], wb[RL], vt[RL], vb[RL];
    double ss = 0.0;
#pragma unroll
    for (int u = 0; u < RL; u++) {
        const int r = g + kJG * u;
        wt[u] = (r < p && ct0 < p) ? T[r + (int64_t)ct0 * ldt] : 0.0;
        wb[u] = (r < p && cb0 < p) ? T[r + (int64_t)cb0 * ldt] : 0.0;
        vt[u] = (r < p && r == ct0) ? 1.0 : 0.0;
        vb[u] = (r < p && r == cb0) ? 1.0 : 0.0;
        ss = fma(wt[u], wt[u], ss);
        ss = fma(wb[u], wb[u], ss);
    }
#pragma unroll
    for (int off = kJG / 2; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (g == 0 && slot) red[q] = ss;
    __syncthreads();
    double tot = 0.0;
    for (int i = 0; i < np2; i++) tot += red[i];  // fixed order
    const double tiny = (double)p * 2.220446049250313e-16 * sqrt(tot);
    const double tiny2 = tiny * tiny, ctol2 = ctol * ctol;
    // positions moving into the slot's two positions (read side of the exchange)
    const int srct = q == 0 ? 0 : (q == 1 ? pe - 1 : q - 1), srcb = pe - 2 - q;
    int buf = 0, sweep;
    bool conv = false;
    for (sweep = 1; sweep <= max_sweeps; sweep++) {
        int rot = 0, any = 0;
        int gt = ct0, gb = cb0;  // columns at the slot's positions in round r
        for (int r = 0; r < m; r++) {
            const bool live = gt < p && gb < p;
            const bool tlow = gt < gb;
            // sums branch-free (the 4 groups of a warp differ in orientation;
            // shuffles under divergence are serialized), then oriented
            double st2, sb2, gam;
            group_pair_sums<RL>(wt, wb, st2, sb2, gam);
            const double al = tlow ? st2 : sb2, be = tlow ? sb2 : st2;
            if (live && al > tiny2 && be > tiny2 && gam * gam > ctol2 * (al * be)) {
                double c, s;
                rot_cs(jacobi_tan(al, be, gam), c, s);
                // (A, B) = (lower, higher): A' = c A - s B, B' = s A + c B; with the
                // top column the higher one, the same form with s -> -s
                const double sx = tlow ? s : -s;
#pragma unroll
                for (int u = 0; u < RL; u++) {
                    const double x = wt[u], y = wb[u];
                    wt[u] = c * x - sx * y;
                    wb[u] = sx * x + c * y;
                    const double vx = vt[u], vy = vb[u];
                    vt[u] = c * vx - sx * vy;
                    vb[u] = sx * vx + c * vy;
                }
                rot = 1;
            }
            if (m > 1) {
                double *B = xs + (size_t)buf * pe * PS;
                if (slot) {
                    double *st = B + (size_t)q * PS + g, *sb = B + (size_t)(pe - 1 - q) * PS + g;
#pragma unroll
                    for (int u = 0; u < RL; u++) {
                        st[kJG * u] = wt[u];
                        st[R + kJG * u] = vt[u];
                        sb[kJG * u] = wb[u];
                        sb[R + kJG * u] = vb[u];
                    }
                }
                if (r == m - 1) any = __syncthreads_or(rot);
                else __syncthreads();
                if (slot) {
                    const double *lt = B + (size_t)srct * PS + g, *lb = B + (size_t)srcb * PS + g;
#pragma unroll
                    for (int u = 0; u < RL; u++) {
                        if (q != 0) {
                            wt[u] = lt[kJG * u];
                            vt[u] = lt[R + kJG * u];
                        }
                        wb[u] = lb[kJG * u];
                        vb[u] = lb[R + kJG * u];
                    }
                }
                buf ^= 1;
            } else {
                any = __syncthreads_or(rot);
            }
            // next round: every column one position on (position 0 fixed)
            if (q != 0) gt = (gt == 1) ? m : gt - 1;
            gb = (gb == 1) ? m : gb - 1;
        }
        if (!any) {
            conv = true;
            break;
        }
    }
#pragma unroll
    for (int u = 0; u < RL; u++) {
        const int r = g + kJG * u;
        if (r < p) {
            if (ct0 < p) {
                Wout[r + (int64_t)ct0 * p] = wt[u];
                Vout[r + (int64_t)ct0 * p] = vt[u];
            }
            if (cb0 < p) {
                Wout[r + (int64_t)cb0 * p] = wb[u];
                Vout[r + (int64_t)cb0 * p] = vb[u];
            }
        }
    }
    if (threadIdx.x == 0) {
        ctrl->svd_tiny = tiny;
        ctrl->svd_sweeps = conv ? sweep : max_sweeps;
        ctrl->svd_status = conv ? 0 : (int)SVDSC_ESVD_NOCONV;
    }
}

// V = J_1 J_2 ... (the logged rotations) for R rows of V per CTA: row r of V is
// e_r^T J_1 J_2 ..., independent of the other rows.  Thread (q, i) applies
// rotation q of every round to row i of the CTA's R rows (rotations of one
// round touch disjoint columns).  The log is staged through shared memory in
// chunks of kLogRounds rounds with cp.async double buffering; (c, s) come
// from the log, so V sees exactly the rotations applied to W.
__global__ void k_apply_log(int p, int per_round, int rounds_per_sweep, const RotLog *__restrict__ rlog,
                            const Ctrl *ctrl, double *V, int R, int kLogRounds, const int *abort) {
    if (aborted(abort)) return;
    extern __shared__ double sm[];
    const int64_t total_rounds = (int64_t)ctrl->svd_sweeps * rounds_per_sweep;
    double *rows = sm;                                                 // R x p
    RotLog *buf = reinterpret_cast<RotLog *>(rows + (((int64_t)R * p + 1) & ~1));  // 2 x kLogRounds x per_round
    const int chunk = kLogRounds * per_round;
    const int r0 = blockIdx.x * R;
    for (int idx = threadIdx.x; idx < R * p; idx += blockDim.x) {
        const int i = idx / p, j = idx % p;
        rows[idx] = (r0 + i == j) ? 1.0 : 0.0;
    }
    auto load_chunk = [&](int64_t first_round, RotLog *dst) {
        const int64_t nrem = total_rounds - first_round;
        const int n16 = (int)min((int64_t)kLogRounds, max((int64_t)0, nrem)) * per_round * 2;  // 16-byte units
        const char *src = reinterpret_cast<const char *>(rlog + first_round * per_round);
        for (int i = threadIdx.x; i < n16; i += blockDim.x) {
            const unsigned saddr = (unsigned)__cvta_generic_to_shared(reinterpret_cast<char *>(dst) + 16 * i);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(src + 16 * i));
        }
        asm volatile("cp.async.commit_group;");
    };
    if (total_rounds > 0) load_chunk(0, buf);
    const int q = threadIdx.x % per_round, i = threadIdx.x / per_round;
    const bool act = i < R;
    double *row = rows + i * p;
    int cur = 0;
    for (int64_t base = 0; base < total_rounds; base += kLogRounds) {
        if (base + kLogRounds < total_rounds) {
            load_chunk(base + kLogRounds, buf + (cur ^ 1) * chunk);
            asm volatile("cp.async.wait_group 1;");
        } else {
            asm volatile("cp.async.wait_group 0;");
        }
        __syncthreads();
        const RotLog *lg = buf + cur * chunk;
        const int nr = (int)min((int64_t)kLogRounds, total_rounds - base);
        for (int k = 0; k < nr; k++) {
            if (act) {
                const RotLog &e = lg[k * per_round + q];
                const double c = e.c, s = e.s;
                if (c != 0.0) {
                    const double x = row[e.a], y = row[e.b];
                    row[e.a] = c * x - s * y;
                    row[e.b] = s * x + c * y;
                }
            }
            __syncthreads();
        }
        cur ^= 1;
    }
    for (int idx = threadIdx.x; idx < R * p; idx += blockDim.x) {
        const int ii = idx / p, j = idx % p;
        if (r0 + ii < p) V[(r0 + ii) + (int64_t)j * p] = rows[idx];
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
    __shared__ double sorted[kMaxP];  // Sh in shared memory (the completion scan reads it)
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
        if (lane == 0) {
            Sh[d] = sj;
            sorted[d] = sj;
        }
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
            if (sorted[d] > 0.0) continue;
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

// ---------------------------------------------------------------------------
// Recombination on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64):
// Qout(:, 0:k) = Q(:, 0:t) W(:, 0:k), a (N x t)(t x k) contraction at
// 19-38 flop/B, so it is FP64-throughput bound, not HBM
// bound.  A CTA owns a 32-row tile: the whole tile Q(r0:r0+32, 0:t) is staged
// in shared memory (cp.async) before any output row is written, which makes the
// in-place call (Qout == Q) safe.  W streams through shared memory in chunks of
// kRC rows (register-staged prefetch of chunk c+1 during chunk c).  Four warps:
// warp (mh, nh) computes rows 16 mh .. 16 mh + 15 (two m8 tiles) times n8 tiles
// nh*NTW .. nh*NTW + NTW - 1.  Fragment layout of m8n8k4 (PTX ISA): A row =
// lane/4, col = lane%4; B row = lane%4, col = lane/4; C row = lane/4, cols
// 2(lane%4) + {0, 1}.  Shared strides are 4 mod 16 doubles, so every fragment
// load of a half-warp hits 16 distinct banks.
constexpr int kRT = 32;       // rows per tile
constexpr int kLDT = kRT + 4; // tile stride (doubles)
constexpr int kRC = 8;        // W rows per chunk (two k4 steps)

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int NTW>
__global__ void __launch_bounds__(128) k_recombine_dmma(int64_t N, int t, int k, const double *Q, int64_t ldq,
                                                        const double *__restrict__ Wm, int ldw, double *Qout,
                                                        int64_t ldo, int ldws, bool vec) {
    extern __shared__ __align__(16) double sm_rc[];
    const int KP = (t + kRC - 1) / kRC * kRC;
    double *tile = sm_rc;                      // KP x kLDT  (tile[j * kLDT + row])
    double *wsb = tile + (size_t)KP * kLDT;    // 2 x kRC x ldws (wsb[l * ldws + col])
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int mh = wid & 1, nh = wid >> 1;
    const int g = lane >> 2, tg = lane & 3;
    const int NT = (k + 7) >> 3;
    const int nch = KP / kRC;
    const int wpc = kRC * NT * 8;              // W elements per chunk (incl. padding columns)
    constexpr int kWReg = (kRC * 2 * NTW * 8 + 127) / 128;
    // zero the K padding rows of the tile once (never overwritten)
    for (int idx = tid; idx < (KP - t) * kLDT; idx += 128) tile[(size_t)t * kLDT + idx] = 0.0;
    const int64_t ntiles = (N + kRT - 1) / kRT;
    double wr[kWReg];
    auto wload = [&](int c) {  // chunk c of W into registers (zero beyond t / k)
#pragma unroll
        for (int u = 0; u < kWReg; u++) {
            const int idx = tid + 128 * u;
            double x = 0.0;
            if (idx < wpc) {
                const int l = idx % kRC, j = idx / kRC;
                const int lg = c * kRC + l;
                if (lg < t && j < k) x = __ldg(Wm + lg + (int64_t)j * ldw);
            }
            wr[u] = x;
        }
    };
    auto wstore = [&](int buf) {
        double *dst = wsb + (size_t)buf * kRC * ldws;
#pragma unroll
        for (int u = 0; u < kWReg; u++) {
            const int idx = tid + 128 * u;
            if (idx < wpc) dst[(idx % kRC) * ldws + idx / kRC] = wr[u];
        }
    };
    for (int64_t tI = blockIdx.x; tI < ntiles; tI += gridDim.x) {
        const int64_t r0 = tI * kRT;
        const int nr = (int)min((int64_t)kRT, N - r0);
        if (vec && nr == kRT) {
            for (int idx = tid; idx < t * (kRT / 2); idx += 128) {
                const int j = idx / (kRT / 2), q = (idx % (kRT / 2)) * 2;
                const unsigned sa = (unsigned)__cvta_generic_to_shared(tile + (size_t)j * kLDT + q);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(Q + r0 + q + (int64_t)j * ldq));
            }
            asm volatile("cp.async.commit_group;");
        } else {
            for (int idx = tid; idx < t * kRT; idx += 128) {
                const int j = idx / kRT, q = idx % kRT;
                tile[(size_t)j * kLDT + q] = q < nr ? Q[r0 + q + (int64_t)j * ldq] : 0.0;
            }
        }
        wload(0);
        wstore(0);
        asm volatile("cp.async.wait_group 0;");
        __syncthreads();
        double acc[2][NTW][2];
#pragma unroll
        for (int i = 0; i < 2; i++)
#pragma unroll
            for (int n = 0; n < NTW; n++) acc[i][n][0] = acc[i][n][1] = 0.0;
        for (int c = 0; c < nch; c++) {
            if (c + 1 < nch) wload(c + 1);
            const double *wb = wsb + (size_t)(c & 1) * kRC * ldws;
#pragma unroll
            for (int ks = 0; ks < kRC / 4; ks++) {
                const int kk = c * kRC + ks * 4 + tg;
                const double a0 = tile[(size_t)kk * kLDT + mh * 16 + g];
                const double a1 = tile[(size_t)kk * kLDT + mh * 16 + 8 + g];
#pragma unroll
                for (int n = 0; n < NTW; n++) {
                    const int nt = nh * NTW + n;
                    if (nt < NT) {
                        const double b = wb[(ks * 4 + tg) * ldws + nt * 8 + g];
                        dmma(acc[0][n][0], acc[0][n][1], a0, b);
                        dmma(acc[1][n][0], acc[1][n][1], a1, b);
                    }
                }
            }
            if (c + 1 < nch) wstore((c + 1) & 1);
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int row = mh * 16 + i * 8 + g;
            if (row < nr) {
#pragma unroll
                for (int n = 0; n < NTW; n++) {
                    const int col = (nh * NTW + n) * 8 + tg * 2;
                    if (col < k) Qout[r0 + row + (int64_t)col * ldo] = acc[i][n][0];
                    if (col + 1 < k) Qout[r0 + row + (int64_t)(col + 1) * ldo] = acc[i][n][1];
                }
            }
        }
        __syncthreads();  // the tile buffer is reloaded next iteration
    }
}

}  // namespace

namespace {
// cluster size and half-block width for p columns (0 if W does not fit)
void jacobi_geometry(int p, int &C, int &h) {
    // <= 20 pairs (one warp each) per CTA, W half-blocks resident in shared memory.
    // A round is bound by instruction issue of its pair warps, so more CTAs with
    // fewer pairs each win until the per-sweep cluster exchanges dominate:
    // at least h <= kJMaxH columns per half-block (SVDSC_JACOBI_H overrides).
    const int pe = p + (p & 1);
    int hmax = kJThreads / 32;
    hmax = std::min(hmax, kJMaxH);
    for (C = 1; C <= 16; C <<= 1) {
        h = (pe + 2 * C - 1) / (2 * C);
        if (h <= hmax && (size_t)2 * h * p * 8 <= 210 * 1024 && h * p <= kExR * kJThreads &&
            p <= 32 * kMaxRPL)
            return;
    }
    // fall back to the widest half-blocks if the preferred width does not fit
    for (C = 1; C <= 16; C <<= 1) {
        h = (pe + 2 * C - 1) / (2 * C);
        if (h <= kJThreads / 32 && (size_t)2 * h * p * 8 <= 210 * 1024 && h * p <= kExR * kJThreads &&
            p <= 32 * kMaxRPL)
            return;
    }
    C = 0;
    h = 0;
}
}  // namespace

template <int R>
cudaError_t launch_jacobi(int C, int p, int h, size_t smem, double *W, RotLog *rlog, Ctrl *ctrl, const int *abort,
                          double ctol, cudaStream_t s) {
    if (C == 1) {
        cudaFuncSetAttribute(k_jacobi_block<false, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        k_jacobi_block<false, R><<<1, kJThreads, smem, s>>>(p, h, W, W, rlog, 50, ctrl, abort, ctol, 0);
        return cudaGetLastError();
    }
    // bulk-copy exchange when the second buffer set fits and the half-blocks
    // (h p doubles) are whole 16-byte units (cp.async.bulk alignment), else a
    // register pull
    const int use_bulk = (2 * smem <= 210 * 1024 && (h * p) % 2 == 0) ? 1 : 0;
    if (use_bulk) smem *= 2;
    cudaFuncSetAttribute(k_jacobi_block<true, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (C > 8) cudaFuncSetAttribute(k_jacobi_block<true, R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kJThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // V is replayed from the rotation log by k_apply_log after this launch.  (Round 1
    // replayed it from extra clusters of the same cooperative launch that polled the
    // Jacobi cluster's progress; that result changed under ncu -- a cross-cluster
    // spin protocol inside one launch -- so it was removed.)
    return cudaLaunchKernelEx(&cfg, k_jacobi_block<true, R>, p, h, (const double *)W, W, rlog, 50, ctrl, abort, ctol,
                              use_bulk);
}

size_t small_svd_log_doubles(int p) {
    int C, h;
    jacobi_geometry(p, C, h);
    if (!C) return 1;
    const int64_t per_sweep = jacobi_rounds_per_sweep(C, h) * C * h;
    return (size_t)(50 * per_sweep * (sizeof(RotLog) / sizeof(double)));
}

void small_svd(int p, const double *Tsrc, int ldt, double *W, double *Vw, double *Uh, double *Sh, double *Vh,
               int kneed, Ctrl *ctrl, const int *abort, double *tlog, cudaStream_t s) {
    const double ctol = 2.0 * (double)p * 2.220446049250313e-16;  // reading Q10a
    const int pol = g_policy.small_svd;  // SVDSC_POLICY_SMALL_SVD
    if (p <= 64 && (pol == 0 || pol == 2)) {
        // register Jacobi: one launch for W and V, then the finish
        const int pe = p + (p & 1);
        const int threads = ((pe / 2) * kJG + 31) / 32 * 32;
        const size_t smem = (size_t)2 * pe * (2 * kJG * (p <= 32 ? 4 : 8) + 8) * sizeof(double);
        if (p <= 32) {
            k_jacobi_reg<4><<<1, threads, smem, s>>>(p, Tsrc, ldt, W, Vw, ctrl, abort, ctol, 50);
        } else {
            cudaFuncSetAttribute(k_jacobi_reg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_jacobi_reg<8><<<1, threads, smem, s>>>(p, Tsrc, ldt, W, Vw, ctrl, abort, ctol, 50);
        }
        count_launch();
        k_svd_finish<<<1, 1024, 0, s>>>(p, W, Vw, Uh, Sh, Vh, kneed, ctrl, abort);
        count_launch();
        return;
    }
    k_copy_T<<<1, 1024, 0, s>>>(p, Tsrc, ldt, W, Vw, ctrl, abort);
    count_launch();
    if (pol == 1) tlog = nullptr;  // one-CTA Jacobi
    bool done = false;
    int C, h;
    jacobi_geometry(p, C, h);
    if (tlog && C) {
        RotLog *rlog = reinterpret_cast<RotLog *>(tlog);
        const size_t smem = (size_t)2 * h * p * 8;
        cudaError_t e;
        const int rpl = (p + 31) / 32;
        e = rpl <= 1 ? launch_jacobi<1>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 2 ? launch_jacobi<2>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 3 ? launch_jacobi<3>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 4 ? launch_jacobi<4>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 5 ? launch_jacobi<5>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 6 ? launch_jacobi<6>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 8 ? launch_jacobi<8>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 10 ? launch_jacobi<10>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 12 ? launch_jacobi<12>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
          : rpl <= 16 ? launch_jacobi<16>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s)
                      : launch_jacobi<20>(C, p, h, smem, W, rlog, ctrl, abort, ctol, s);
        if (e == cudaSuccess) {
            count_launch();
            const int per_round = C * h;
            const int rps = (int)jacobi_rounds_per_sweep(C, h);
            const int R = std::max(1, std::min(8, 1024 / per_round));
            const int threads = ((per_round * R + 31) / 32) * 32;
            const size_t rows_b = (size_t)(R * p + 2) * 8;
            const int lrc = (int)std::max<size_t>(1, std::min<size_t>(16, (200 * 1024 - rows_b) / (2 * per_round * sizeof(RotLog))));
            const size_t smem2 = rows_b + 2 * (size_t)lrc * per_round * sizeof(RotLog);
            cudaFuncSetAttribute(k_apply_log, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
            k_apply_log<<<(p + R - 1) / R, threads, smem2, s>>>(p, per_round, rps, rlog, ctrl, Vw, R, lrc, abort);
            count_launch();
            done = true;
        } else {
            cudaGetLastError();  // clear and fall back
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

template <int NTW>
bool launch_recombine_dmma(int64_t N, int t, int k, const double *Q, int64_t ldq, const double *W, int ldw,
                           double *Qout, int64_t ldo, int nsm, cudaStream_t s) {
    const int NT = (k + 7) / 8;
    const int KP = (t + kRC - 1) / kRC * kRC;
    const int ldws = (NT * 8 + 15) / 16 * 16 + 4;
    const size_t smem = ((size_t)KP * kLDT + 2 * (size_t)kRC * ldws) * sizeof(double);
    if (smem > 220 * 1024) return false;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_recombine_dmma<NTW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr = true;
    }
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_recombine_dmma<NTW>, 128, smem);
    if (bps < 1) return false;
    const bool vec = (ldq % 2 == 0) && ((reinterpret_cast<uintptr_t>(Q) & 15) == 0);
    const int64_t ntiles = (N + kRT - 1) / kRT;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)nsm * bps));
    k_recombine_dmma<NTW><<<grid, 128, smem, s>>>(N, t, k, Q, ldq, W, ldw, Qout, ldo, ldws, vec);
    count_launch();
    return true;
}

void recombine(int64_t N, int t, int k, const double *Q, int64_t ldq, const double *W, int ldw, double *Qout,
               int64_t ldo, int nsm, cudaStream_t s) {
    {
        const int ntw = ((k + 7) / 8 + 1) / 2;
        bool ok = false;
        if (ntw <= 1) ok = launch_recombine_dmma<1>(N, t, k, Q, ldq, W, ldw, Qout, ldo, nsm, s);
        else if (ntw <= 2) ok = launch_recombine_dmma<2>(N, t, k, Q, ldq, W, ldw, Qout, ldo, nsm, s);
        else if (ntw <= 4) ok = launch_recombine_dmma<4>(N, t, k, Q, ldq, W, ldw, Qout, ldo, nsm, s);
        else if (ntw <= 7) ok = launch_recombine_dmma<7>(N, t, k, Q, ldq, W, ldw, Qout, ldo, nsm, s);
        else if (ntw <= 13) ok = launch_recombine_dmma<13>(N, t, k, Q, ldq, W, ldw, Qout, ldo, nsm, s);
        if (ok) return;
    }
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
