// matvec.cu -- the two products of every Lanczos step:
//   a1: w = A^T u_i - alpha_i v_i   (Alg. 1 line 5)
//   a5: z = A v_{i+1} - beta_i u_i  (Alg. 1 line 7)
// The paper calls MKL_dcsrmv / an OpenMP SpMV and cblas_dgemv for
// dense A.  Here:
//   * CSR SpMV with rows binned by length: sub-warp "vector" groups of 2..32
//     lanes, CTA-per-row, and multi-CTA chunks for rows > kLongRow nnz; every
//     row sum is a fixed-shape tree, so results are run-to-run deterministic.
//   * A^T u runs the same SpMV on a device-built CSC copy (= CSR of A^T) whose
//     in-column order is by row, i.e. the oracle's accumulation order.
//   * dense GEMV N/T: 128-bit coalesced loads of the column-major A, split over
//     columns (N) or rows (T) into a grid of ~8 CTAs per SM, deterministic
//     split-K reduction fused with the epilogue.
// All kernels are HBM-bandwidth bound; the epilogue (- c * yprev) is fused.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.h"

namespace svdsc {

thread_local int64_t g_launches = 0;
thread_local Policy g_policy;
thread_local cudaMemPool_t g_pool = nullptr;
thread_local cudaStream_t g_pool_stream = nullptr;

void *analysis_alloc(size_t bytes) {
    void *p = nullptr;
    bytes = std::max<size_t>(bytes, 8);
    const cudaError_t e = g_pool ? cudaMallocFromPoolAsync(&p, bytes, g_pool, g_pool_stream) : cudaMalloc(&p, bytes);
    if (e != cudaSuccess) throw std::runtime_error(std::string("analysis allocation: ") + cudaGetErrorString(e));
    return p;
}
void analysis_free(void *p) {
    if (!p) return;
    if (g_pool) cudaFreeAsync(p, g_pool_stream);
    else cudaFree(p);
}

namespace {

constexpr int kLongRow = 65536;   // rows longer than this are split into chunks

__device__ __forceinline__ bool aborted(const int *abort) {
    return abort != nullptr && *(volatile const int *)abort != 0;
}

// bin of a row of length L: 0..4 = vector groups of 2,4,8,16,32 lanes,
// 5 = CTA per row, 6 = long (chunked)
__host__ __device__ __forceinline__ int row_bin(int64_t L) {
    if (L <= 4) return 0;
    if (L <= 8) return 1;
    if (L <= 16) return 2;
    if (L <= 64) return 3;
    if (L <= 2048) return 4;
    if (L <= kLongRow) return 5;
    return 6;
}

// row counts per bin (cnt[0..7]) and the longest row (cnt[8])
__global__ void k_bin_count(int64_t nrows, const int64_t *__restrict__ rp, unsigned long long *cnt) {
    __shared__ unsigned int sc[8];
    __shared__ unsigned long long smax;
    if (threadIdx.x < 8) sc[threadIdx.x] = 0;
    if (threadIdx.x == 0) smax = 0;
    __syncthreads();
    unsigned long long mx = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t L = rp[r + 1] - rp[r];
        atomicAdd(&sc[row_bin(L)], 1u);
        mx = max(mx, (unsigned long long)L);
    }
    atomicMax(&smax, mx);
    __syncthreads();
    if (threadIdx.x < 8 && sc[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], (unsigned long long)sc[threadIdx.x]);
    if (threadIdx.x == 0) atomicMax(&cnt[8], smax);
}

// lengths of the listed rows (the long-row table: one D2H instead of one per row)
__global__ void k_row_len(int64_t n, const int32_t *__restrict__ rows, const int64_t *__restrict__ rp, int64_t *len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) len[i] = rp[rows[i] + 1] - rp[rows[i]];
}

// bin key and row id per row; a stable radix sort by key then lists every bin's
// rows in ascending order (streaming access to row_ptr / col / val / y)
__global__ void k_bin_keys(int64_t nrows, const int64_t *__restrict__ rp, uint8_t *key, int32_t *ids) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        key[r] = (uint8_t)row_bin(rp[r + 1] - rp[r]);
        ids[r] = (int32_t)r;
    }
}

// y[row] = sum - c*yprev[row]
__device__ __forceinline__ void epilogue_store(double *y, int64_t r, double sum, double c,
                                               const double *yprev) {
    if (yprev) sum -= c * yprev[r];
    y[r] = sum;
}

// G lanes per row; the whole warp iterates in lock-step so full-mask shuffles
// are legal.  Each lane issues kU index/value loads (streaming, evict-first: A
// is read once per product) before their kU dependent x gathers (read-only
// path, L1/L2 resident), so a warp keeps 2 kU + kU loads in flight instead of a
// serial load -> gather -> FMA chain.  rows == nullptr: the bin is the identity
// (every row, in order).  Fixed shape per G: deterministic.
template <int G, int kU>
__device__ __forceinline__ void spmv_vec_rows(const int32_t *__restrict__ rows, int64_t count,
                                                  const int64_t *__restrict__ rp,
                                                  const int32_t *__restrict__ col,
                                                  const double *__restrict__ val,
                                                  const double *__restrict__ x, double *__restrict__ y,
                                                  const double *c_dev, const double *__restrict__ yprev,
                                                  int64_t blk, int64_t nblk) {
    constexpr int GPW = kWarp / G;  // groups per warp
    const int lane = threadIdx.x & 31;
    const int sub = lane % G;
    const int64_t warp_g = (blk * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (nblk * blockDim.x) >> 5;
    const double c = c_dev ? *c_dev : 0.0;
    for (int64_t base = warp_g * GPW; base < count; base += nwarps * GPW) {
        const int64_t g = base + lane / G;
        double sum = 0.0;
        int64_t r = -1;
        if (g < count) {
            r = rows ? (int64_t)rows[g] : g;
            const int64_t p0 = rp[r], p1 = rp[r + 1];
            double s1 = 0.0;
            for (int64_t p = p0 + sub; p < p1; p += G * kU) {
                int ci[kU];
                double vv[kU], xv[kU];
#pragma unroll
                for (int u = 0; u < kU; u++) {
                    const int64_t q = p + (int64_t)u * G;
                    const bool ok = q < p1;
                    ci[u] = ok ? __ldcs(col + q) : 0;
                    vv[u] = ok ? __ldcs(val + q) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kU; u++) xv[u] = __ldg(x + ci[u]);
#pragma unroll
                for (int u = 0; u < kU; u += 2) {
                    sum = fma(vv[u], xv[u], sum);
                    s1 = fma(vv[u + 1], xv[u + 1], s1);
                }
            }
            sum += s1;
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off, G);
        if (sub == 0 && r >= 0) epilogue_store(y, r, sum, c, yprev);
    }
}


// All vector bins in ONE launch: CTAs [bstart[b], bstart[b+1]) serve bin b
// with its group width (2, 4, 8, 16, 32 lanes per row).  Avoids one
// serialized (and often tiny) launch per non-empty bin.
// group shape (lanes per row, loads in flight per lane) of bins 3 and 4
// (compile-time tunables: -DSVDSC_BIN3_G=... etc.)
#ifndef SVDSC_BIN3_G
#define SVDSC_BIN3_G 8
#define SVDSC_BIN3_U 8
#endif
#ifndef SVDSC_BIN4_G
#define SVDSC_BIN4_G 16
#define SVDSC_BIN4_U 8
#endif
constexpr int kBin3G = SVDSC_BIN3_G, kBin3U = SVDSC_BIN3_U;
constexpr int kBin4G = SVDSC_BIN4_G, kBin4U = SVDSC_BIN4_U;

struct BinArgs {
    const int32_t *rows[5];  // nullptr: identity bin
    int64_t count[5];
    int bstart[6];
};

__global__ void __launch_bounds__(256) k_spmv_bins(BinArgs ba, const int64_t *__restrict__ rp,
                                                   const int32_t *__restrict__ col, const double *__restrict__ val,
                                                   const double *__restrict__ x, double *__restrict__ y,
                                                   const double *c_dev, const double *__restrict__ yprev,
                                                   const int *abort) {
    pdl_wait();  // launched with launch_pdl: x is the predecessor's output
    pdl_trigger();
    if (aborted(abort)) return;
    const int bx = blockIdx.x;
    int b = 0, lo = ba.bstart[0], hi = ba.bstart[1];
#pragma unroll
    for (int q = 1; q < 5; q++)
        if (bx >= ba.bstart[q]) {
            b = q;
            lo = ba.bstart[q];
            hi = ba.bstart[q + 1];
        }
    const int64_t blk = bx - lo, nblk = hi - lo;
    switch (b) {
        // (lanes per row, loads in flight per lane): rows of 17-64 nnz take 8 lanes x 8
        // (one pass for up to 64 nnz, 4 rows per warp), 65-2048 take 16 x 8 -- measured
        // best of the tried shapes (config 3: 53.5 vs 58 us; config 4 A^T: 798 vs 868 us)
        case 0: spmv_vec_rows<2, 4>(ba.rows[0], ba.count[0], rp, col, val, x, y, c_dev, yprev, blk, nblk); break;
        case 1: spmv_vec_rows<4, 4>(ba.rows[1], ba.count[1], rp, col, val, x, y, c_dev, yprev, blk, nblk); break;
        case 2: spmv_vec_rows<8, 4>(ba.rows[2], ba.count[2], rp, col, val, x, y, c_dev, yprev, blk, nblk); break;
        case 3: spmv_vec_rows<kBin3G, kBin3U>(ba.rows[3], ba.count[3], rp, col, val, x, y, c_dev, yprev, blk, nblk); break;
        default: spmv_vec_rows<kBin4G, kBin4U>(ba.rows[4], ba.count[4], rp, col, val, x, y, c_dev, yprev, blk, nblk); break;
    }
}

__device__ __forceinline__ double block_sum_256(double v, double *sh /* >= 8 */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += sh[i];
    return s;  // valid on thread 0
}

// one CTA per row (rows of 2k..64k nnz)
__global__ void __launch_bounds__(256) k_spmv_cta(const int32_t *__restrict__ rows, int64_t count,
                                                  const int64_t *__restrict__ rp,
                                                  const int32_t *__restrict__ col,
                                                  const double *__restrict__ val,
                                                  const double *__restrict__ x, double *__restrict__ y,
                                                  const double *c_dev, const double *__restrict__ yprev,
                                                  const int *abort) {
    if (aborted(abort)) return;
    __shared__ double sh[8];
    const double c = c_dev ? *c_dev : 0.0;
    for (int64_t g = blockIdx.x; g < count; g += gridDim.x) {
        const int32_t r = rows[g];
        const int64_t p0 = rp[r], p1 = rp[r + 1];
        double sum = 0.0;
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) sum = fma(val[p], __ldg(x + col[p]), sum);
        sum = block_sum_256(sum, sh);
        if (threadIdx.x == 0) epilogue_store(y, r, sum, c, yprev);
    }
}

// chunks of long rows: partial[ch] = sum over the chunk
__global__ void __launch_bounds__(256) k_spmv_chunks(int64_t n_chunks, const int32_t *__restrict__ chunk_row,
                                                     const int64_t *__restrict__ chunk_first,
                                                     const int32_t *__restrict__ long_rows,
                                                     const int64_t *__restrict__ rp,
                                                     const int32_t *__restrict__ col,
                                                     const double *__restrict__ val,
                                                     const double *__restrict__ x, double *partial,
                                                     const int *abort) {
    if (aborted(abort)) return;
    __shared__ double sh[8];
    for (int64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
        const int32_t slot = chunk_row[ch];
        const int32_t r = long_rows[slot];
        const int64_t k = ch - chunk_first[slot];
        const int64_t p0 = rp[r] + k * kLongRow;
        const int64_t p1 = min(rp[r + 1], p0 + (int64_t)kLongRow);
        double sum = 0.0;
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) sum = fma(val[p], __ldg(x + col[p]), sum);
        sum = block_sum_256(sum, sh);
        if (threadIdx.x == 0) partial[ch] = sum;
    }
}

__global__ void k_spmv_chunks_fix(int64_t n_long, const int32_t *__restrict__ long_rows,
                                  const int64_t *__restrict__ chunk_first, const double *partial,
                                  double *y, const double *c_dev, const double *yprev, const int *abort) {
    if (aborted(abort)) return;
    const double c = c_dev ? *c_dev : 0.0;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_long;
         s += (int64_t)gridDim.x * blockDim.x) {
        double sum = 0.0;
        for (int64_t ch = chunk_first[s]; ch < chunk_first[s + 1]; ch++) sum += partial[ch];
        epilogue_store(y, long_rows[s], sum, c, yprev);
    }
}


// ---------------------------------------------------------------------------
// Register-segmented SpMV ("seg", the default schedule for every CSR operand:
// A and its CSC copy, uniform and power-law rows alike).  The nonzeros are cut
// into chunks of kSegChunk = 32 lanes x 8 consecutive nonzeros; each warp of a
// persistent grid owns a contiguous run of chunks (nnz-balanced, whatever the
// row lengths).  Per chunk a lane loads its 8 column indices and values with
// 128-bit streaming loads, issues its 8 independent x gathers, and sums its
// products in order, splitting them at row starts read from a bitmap (1 bit per
// nonzero, built at analysis): rows wholly inside the lane are finished there;
// the pieces that cross lanes are joined by a segmented suffix sum over the
// warp (5 shuffles), the piece that crosses chunks is carried in a register.
// Rows crossing warp ranges leave partial sums (head / tail per range) that the
// last CTA to finish adds in range order.  No shared memory, no barriers in
// the loop (round 1's nnz-tile kernel spent ~1/3 of its L1 cycles on shared-
// memory staging and bank conflicts); every sum has a fixed order, so the
// result is bitwise reproducible.  The row index of the k-th row start is
// rows[k] (non-empty rows, ascending); cstart[ch] = row starts before chunk ch.
struct SegArgs {
    int64_t nnz;
    int nchunks, cpw, nranges;
    const int32_t *col;
    const double *val;
    const double *x;
    const uint32_t *bits;
    const int32_t *rows, *cstart, *empty;
    int64_t nempty;
    double *y;
    const double *c_dev, *yprev;
    double *head, *tail;
    unsigned int *flag;  // per warp range: 1 once its head / tail piece is published (the joiner resets it)
    const int *abort;
};
constexpr int kSegThreads = 256;
constexpr unsigned kFull = 0xffffffffu;
#ifndef SVDSC_SEG_MINB
#define SVDSC_SEG_MINB 5
#endif
#ifndef SVDSC_SEG_FULLPF
#define SVDSC_SEG_FULLPF 0
#endif
constexpr bool kSegFullPf = SVDSC_SEG_FULLPF != 0;
constexpr int kSegMinBlocks = SVDSC_SEG_MINB;

// the first nonzero of warp range w continues a row that began before it
__device__ __forceinline__ bool seg_mid(const SegArgs &a, int w) {
    const int64_t b = (int64_t)w * a.cpw * kSegChunk;
    return b < a.nnz && !((__ldg(a.bits + (b >> 5)) >> (b & 31)) & 1u);
}

__device__ __forceinline__ void seg_store(const SegArgs &a, int k, double s, double c) {
    const int r = __ldg(a.rows + k);
    if (a.yprev) s -= c * a.yprev[r];
    a.y[r] = s;
}

__device__ __forceinline__ void seg_publish(const SegArgs &a, int w) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.flag + w), "r"(1u) : "memory");
}

// Row k began in an earlier warp range and ends in range w with the piece
// `own`: wait for the earlier ranges' pieces (decoupled look-back: only
// lower-numbered ranges, i.e. warps of CTAs dispatched no later than this
// one, are waited for) and add them in range order: tail of the range where
// the row began, heads of the ranges it spans whole, then own.  One lane.
__device__ __forceinline__ void seg_join(const SegArgs &a, int w, int k, double own, double c) {
    int wf = w;
    for (;;) {
        const int wp = wf - 1;
        unsigned f;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.flag + wp) : "memory");
            if (f == 1u) break;
            __nanosleep(64);
        }
        if (wp > 0 && seg_mid(a, wp) && __ldg(a.cstart + wp * a.cpw) - 1 == k) {
            wf = wp;  // range wp lies wholly inside row k: its piece is head[wp]
            continue;
        }
        break;  // row k began in range wp = wf - 1: its piece is tail[wp]
    }
    double s = __ldcg(a.tail + wf - 1);
    for (int j = wf; j < w; j++) s += __ldcg(a.head + j);
    seg_store(a, k, s + own, c);
    // every published piece has exactly one joiner: reset its flag for the
    // next launch (stream order), so no launch counter is needed (graph-safe)
    for (int j = wf - 1; j < w; j++) a.flag[j] = 0u;
}

// one lane's kSegK consecutive nonzeros of a chunk: column indices, row-start
// bits and the chunk's row-start offset (seg_load_ci), values (seg_load_v)
// The chunk's row-start bits are kSegK whole words (the bitmap is padded to
// whole chunks): every lane reads them (one broadcast 128-bit load per 4
// words) and takes its own kSegK bits and the count of starts before them --
// no warp scan for the row-start offsets.
__device__ __forceinline__ void seg_load_ci(const SegArgs &a, int ch, int lane, int (&ci)[kSegK], uint32_t &bits,
                                            int &kb) {
    constexpr uint32_t kMask = (1u << kSegK) - 1u;
    constexpr int kLanesPerWord = 32 / kSegK;
    const int64_t e = (int64_t)ch * kSegChunk + kSegK * lane;
    {
        uint32_t wd[kSegK];
        const uint4 *bp = reinterpret_cast<const uint4 *>(a.bits + (int64_t)ch * kSegK);
#pragma unroll
        for (int q = 0; q < kSegK / 4; q++) {
            const uint4 t = __ldg(bp + q);
            wd[4 * q] = t.x;
            wd[4 * q + 1] = t.y;
            wd[4 * q + 2] = t.z;
            wd[4 * q + 3] = t.w;
        }
        const int myw = lane / kLanesPerWord, sh = kSegK * (lane % kLanesPerWord);
        int before = 0;
        uint32_t mine = 0;
#pragma unroll
        for (int q = 0; q < kSegK; q++) {
            if (q < myw) before += __popc(wd[q]);
            if (q == myw) mine = wd[q];
        }
        bits = (mine >> sh) & kMask;
        kb = __ldg(a.cstart + ch) + before + __popc(mine & ((1u << sh) - 1u));  // starts before this lane
    }
    if (e + kSegK <= a.nnz) {
        const int4 *cp = reinterpret_cast<const int4 *>(a.col + e);
#pragma unroll
        for (int q = 0; q < kSegK / 4; q++) {
            const int4 t = __ldcs(cp + q);
            ci[4 * q] = t.x;
            ci[4 * q + 1] = t.y;
            ci[4 * q + 2] = t.z;
            ci[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < kSegK; u++) ci[u] = e + u < a.nnz ? __ldcs(a.col + e + u) : 0;
    }
}
__device__ __forceinline__ void seg_load_v(const SegArgs &a, int ch, int lane, double (&v)[kSegK]) {
    const int64_t e = (int64_t)ch * kSegChunk + kSegK * lane;
    if (e + kSegK <= a.nnz) {
        const double2 *vp = reinterpret_cast<const double2 *>(a.val + e);
#pragma unroll
        for (int u = 0; u < kSegK / 2; u++) {
            const double2 t = __ldcs(vp + u);
            v[2 * u] = t.x;
            v[2 * u + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < kSegK; u++) v[u] = e + u < a.nnz ? __ldcs(a.val + e + u) : 0.0;
    }
}

__global__ void __launch_bounds__(kSegThreads, kSegMinBlocks) k_spmv_seg(SegArgs a) {
    pdl_wait();  // launched with launch_pdl: x is the predecessor's output
    pdl_trigger();
    if (aborted(a.abort)) return;
    const double c = a.c_dev ? *a.c_dev : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kSegThreads + threadIdx.x; i < a.nempty; i += (int64_t)gridDim.x * kSegThreads) {
        const int r = a.empty[i];
        double s = 0.0;
        if (a.yprev) s -= c * a.yprev[r];
        a.y[r] = s;
    }
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x * (kSegThreads / 32) + (threadIdx.x >> 5);
    if (w < a.nranges) {
        const int c0 = w * a.cpw, c1 = min(a.nchunks, c0 + a.cpw);
        int open = seg_mid(a, w) ? 1 : 0;  // 0 none, 1 began before this range, 2 began in it
        int open_k = __ldg(a.cstart + c0) - 1;
        double carry = 0.0;
        // the piece of the row that began before this range, if it ended here
        // (shared memory, lane 0: keeps the chunk loop's registers free)
        __shared__ double s_pend_own[kSegThreads / 32];
        __shared__ int s_pend_k[kSegThreads / 32];
        const int wl = threadIdx.x >> 5;
        if (lane == 0) s_pend_k[wl] = -1;
        int ci[kSegK];
        double v[kSegK];
        uint32_t bits_n;
        int kb_n;
        seg_load_ci(a, c0, lane, ci, bits_n, kb_n);
        seg_load_v(a, c0, lane, v);
        for (int ch = c0; ch < c1; ch++) {
            double p[kSegK];
#pragma unroll
            for (int u = 0; u < kSegK; u++) p[u] = __ldg(a.x + ci[u]);
            const uint32_t bits = bits_n;
            const int kb = kb_n;
            // the next chunk's index stream is in flight while the gathers return,
            // its value stream while this chunk is reduced and the next gathers issue
            const bool more = ch + 1 < c1;
            if (more) seg_load_ci(a, ch + 1, lane, ci, bits_n, kb_n);
            if constexpr (kSegFullPf) {  // both next streams in flight under the gathers
                double vn[kSegK];
                if (more) seg_load_v(a, ch + 1, lane, vn);
#pragma unroll
                for (int u = 0; u < kSegK; u++) {
                    p[u] *= v[u];
                    v[u] = vn[u];
                }
            } else {
#pragma unroll
                for (int u = 0; u < kSegK; u++) p[u] *= v[u];
                if (more) seg_load_v(a, ch + 1, lane, v);
            }
            // starts before this lane in the chunk (exclusive warp scan of popcounts)
            const int k0 = kb;  // row-start index of the lane's first start
            // in-lane pieces: head (before the first start), finished rows, tail
            double head = 0.0, tl = 0.0;
            int kk = k0;
#pragma unroll
            for (int u = 0; u < kSegK; u++) {
                if ((bits >> u) & 1u) {
                    if (kk > k0) seg_store(a, kk - 1, tl, c);
                    tl = p[u];
                    kk++;
                } else if (kk > k0) {
                    tl += p[u];
                } else {
                    head += p[u];
                }
            }
            const unsigned fmask = __ballot_sync(kFull, bits != 0u);
            // R_l = head_l + (lane l has a start ? 0 : R_{l+1}): segmented suffix sum
            // (Hillis-Steele; the segment flags of a window come from the ballot)
            double R = head;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                double Rn = __shfl_down_sync(kFull, R, off);
                // closed: a start in lanes [lane, lane + off), or the window passes lane 31
                const bool closed = lane + off >= 32 || ((fmask >> lane) & ((1u << off) - 1u)) != 0u;
                if (!closed) R += Rn;
            }
            double Rn1 = __shfl_down_sync(kFull, R, 1);
            if (lane == 31) Rn1 = 0.0;
            // (carry, open and open_k are lane 0's: R_0 is its own R, no broadcast)
            const double piece = tl + Rn1;  // the row begun at this lane's last start, within the chunk
            // that row ends in a later lane of this chunk: finished
            if (bits != 0u && lane < 31 && (fmask >> (lane + 1)) != 0u) seg_store(a, kk - 1, piece, c);
            if (fmask) {
                // the open row ends in this chunk, with the items before its first start
                if (lane == 0) {
                    if (open == 1) {  // joined at the range end (its earlier pieces are published then)
                        s_pend_own[wl] = carry + R;
                        s_pend_k[wl] = open_k;
                    } else if (open == 2) {
                        seg_store(a, open_k, carry + R, c);
                    }
                }
                const int last = 31 - __clz(fmask);
                carry = __shfl_sync(kFull, piece, last);
                open_k = __shfl_sync(kFull, kk - 1, last);
                open = 2;
            } else {
                carry += R;  // (lane 0: R_0, the whole chunk) continues the open row
            }
        }
        if (lane == 0) {
            // publish this range's piece first, then join (no waiting chain
            // across ranges: every range publishes before it waits)
            if (open) {
                const int64_t bend = (int64_t)c1 * kSegChunk;
                const bool ends = bend >= a.nnz || ((__ldg(a.bits + (bend >> 5)) >> (bend & 31)) & 1u);
                if (ends) {
                    if (open == 1) {
                        s_pend_own[wl] = carry;
                        s_pend_k[wl] = open_k;
                    } else {
                        seg_store(a, open_k, carry, c);
                    }
                } else {
                    if (open == 1) a.head[w] = carry;
                    else a.tail[w] = carry;
                    seg_publish(a, w);
                }
            }
            if (s_pend_k[wl] >= 0) seg_join(a, w, s_pend_k[wl], s_pend_own[wl], c);
        }
    }
}

// analysis: row-start bits, non-empty / empty row lists, chunk start counts
__global__ void k_seg_bits(int64_t nrows, const int64_t *__restrict__ rp, uint32_t *bits, int32_t *nzflag) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p0 = rp[r];
        const bool ne = rp[r + 1] > p0;
        if (ne) atomicOr(bits + (p0 >> 5), 1u << (p0 & 31));
        nzflag[r] = ne ? 1 : 0;
    }
}

__global__ void k_seg_rows(int64_t nrows, const int32_t *__restrict__ nzflag, const int32_t *__restrict__ pos,
                           int32_t *rows, int32_t *empty) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        if (nzflag[r]) rows[pos[r]] = (int32_t)r;
        else empty[r - pos[r]] = (int32_t)r;
    }
}

__global__ void k_seg_chunkpop(int64_t nchunks, int64_t nwords, const uint32_t *__restrict__ bits, int32_t *cnt) {
    for (int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ch < nchunks; ch += (int64_t)gridDim.x * blockDim.x) {
        int s = 0;
        for (int q = 0; q < kSegChunk / 32; q++) {
            const int64_t wd = ch * (kSegChunk / 32) + q;
            if (wd < nwords) s += __popc(bits[wd]);
        }
        cnt[ch] = s;
    }
}

// ---------------------------------------------------------------------------
// device CSR -> CSC (CSR of A^T), deterministic: in-column order by (row, position)
__global__ void k_col_count(int64_t nnz, const int32_t *__restrict__ col, int32_t *cnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[col[p]], 1);
}

// exclusive scan of int32 counts into int64 offsets: per-block scan of 1024 items
__global__ void k_scan_block(int64_t n, const int32_t *__restrict__ in, int64_t *out, int64_t *bsum) {
    __shared__ int64_t wsum[32];
    const int64_t i = blockIdx.x * 1024ll + threadIdx.x;
    int64_t v = (i < n) ? in[i] : 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int64_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        int64_t s = wsum[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int64_t o = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += o;
        }
        wsum[lane] = s;  // inclusive warp sums
    }
    __syncthreads();
    int64_t excl = incl - v + (w > 0 ? wsum[w - 1] : 0);
    if (i < n) out[i] = excl;
    if (threadIdx.x == 1023) bsum[blockIdx.x] = excl + v;
}

__global__ void k_scan_add(int64_t n, int64_t *out, const int64_t *boff) {
    const int64_t i = blockIdx.x * 1024ll + threadIdx.x;
    if (i < n) out[i] += boff[blockIdx.x];
}

// warp per row: claim a slot in each column; key = (row << 32) | in-row index
__global__ void k_csc_fill(int64_t nrows, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                           unsigned long long *cursor, uint64_t *key) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < nrows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t p0 = rp[r], p1 = rp[r + 1];
        for (int64_t p = p0 + lane; p < p1; p += 32) {
            unsigned long long pos = atomicAdd(&cursor[col[p]], 1ull);
            key[pos] = ((uint64_t)r << 32) | (uint64_t)(p - p0);
        }
    }
}

// bitonic sort of one segment held in shared memory (n2 = power of two >= len)
__device__ void bitonic_smem(uint64_t *s, int n2) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool up = ((i & k) == 0);
                    uint64_t a = s[i], b = s[ixj];
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}

constexpr int kSegSmem = 4096;  // keys sorted per CTA in shared memory

// segments of length <= kSegSmem: one CTA per segment (grid-stride)
__global__ void __launch_bounds__(256) k_seg_sort(int64_t nseg, const int64_t *__restrict__ off, uint64_t *key) {
    __shared__ uint64_t s[kSegSmem];
    for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
        const int64_t a = off[g], len = off[g + 1] - a;
        if (len <= 1 || len > kSegSmem) continue;
        int n2 = 1;
        while (n2 < len) n2 <<= 1;
        for (int i = threadIdx.x; i < n2; i += blockDim.x) s[i] = (i < len) ? key[a + i] : ~0ull;
        __syncthreads();
        bitonic_smem(s, n2);
        for (int i = threadIdx.x; i < len; i += blockDim.x) key[a + i] = s[i];
        __syncthreads();
    }
}

// sort chunk `blockIdx.x` (kSegSmem keys) of one long segment
__global__ void __launch_bounds__(256) k_chunk_sort(uint64_t *key, int64_t len) {
    __shared__ uint64_t s[kSegSmem];
    const int64_t a = blockIdx.x * (int64_t)kSegSmem;
    const int64_t l = min((int64_t)kSegSmem, len - a);
    for (int i = threadIdx.x; i < kSegSmem; i += blockDim.x) s[i] = (i < l) ? key[a + i] : ~0ull;
    __syncthreads();
    bitonic_smem(s, kSegSmem);
    for (int i = threadIdx.x; i < l; i += blockDim.x) key[a + i] = s[i];
}

// merge sorted runs of width w pairwise by rank (keys are unique)
__global__ void k_merge_runs(const uint64_t *__restrict__ in, uint64_t *out, int64_t len, int64_t w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t run = i / w, pair0 = (run & ~1ll) * w;
        const bool left = (run & 1) == 0;
        const int64_t o0 = left ? pair0 + w : pair0;          // other run start
        const int64_t o1 = min(len, o0 + w);
        const int64_t myrun0 = left ? pair0 : pair0 + w;
        if (o0 >= len) { out[i] = in[i]; continue; }
        const uint64_t v = in[i];
        int64_t lo = o0, hi = o1;  // number of keys < v in the other run
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (in[mid] < v) lo = mid + 1; else hi = mid;
        }
        out[pair0 + (i - myrun0) + (lo - o0)] = v;
    }
}

__global__ void k_csc_gather(int64_t nnz, const uint64_t *__restrict__ key, const int64_t *__restrict__ rp,
                             const double *__restrict__ val, int32_t *tcol, double *tval) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nnz; s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = key[s];
        const int64_t r = (int64_t)(k >> 32);
        const int64_t p = rp[r] + (int64_t)(k & 0xffffffffull);
        tcol[s] = (int32_t)r;
        tval[s] = val[p];
    }
}

inline void check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
T *dev_alloc(CsrOp &op, size_t n) {
    void *p = analysis_alloc(std::max<size_t>(n, 1) * sizeof(T));
    op.owned.push_back(p);
    op.pooled = g_pool != nullptr;
    op.free_stream = g_pool_stream;
    return (T *)p;
}

int grid_for(int64_t work, int threads, int cap = 148 * 16) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

}  // namespace

void csr_free(CsrOp &op) {
    for (void *p : op.owned) {
        if (op.pooled) cudaFreeAsync(p, op.free_stream);
        else cudaFree(p);
    }
    op.owned.clear();
}

namespace {
void seg_analyze(CsrOp &op, cudaStream_t s) {
    const int64_t nrows = op.nrows, nnz = op.nnz;
    const int64_t nchunks0 = std::max<int64_t>(1, (nnz + kSegChunk - 1) / kSegChunk);
    const int64_t nwords = nchunks0 * kSegK;  // whole chunks (the kernel reads a chunk's words at once)
    op.seg_bits = dev_alloc<uint32_t>(op, (size_t)nwords);
    check(cudaMemsetAsync(op.seg_bits, 0, nwords * sizeof(uint32_t), s), "memset");
    int32_t *nzflag = nullptr, *pos = nullptr, *cnt = nullptr;
    nzflag = reinterpret_cast<decltype(nzflag)>(analysis_alloc(std::max<int64_t>(nrows, 1) * sizeof(int32_t)));
    pos = reinterpret_cast<decltype(pos)>(analysis_alloc(std::max<int64_t>(nrows, 1) * sizeof(int32_t)));
    if (nrows > 0) k_seg_bits<<<grid_for(nrows, 256), 256, 0, s>>>(nrows, op.row_ptr, op.seg_bits, nzflag);
    void *tmp = nullptr;
    size_t tb = 0, tb2 = 0;
    const int64_t nchunks = std::max<int64_t>(1, (nnz + kSegChunk - 1) / kSegChunk);
    check(cub::DeviceScan::ExclusiveSum(nullptr, tb, nzflag, pos, (int)std::max<int64_t>(nrows, 1), s), "scan size");
    check(cub::DeviceScan::ExclusiveSum(nullptr, tb2, nzflag, pos, (int)nchunks, s), "scan size");
    tmp = reinterpret_cast<decltype(tmp)>(analysis_alloc(std::max<size_t>({tb, tb2, (size_t)1})));
    int64_t n_nz = 0;
    if (nrows > 0) {
        check(cub::DeviceScan::ExclusiveSum(tmp, tb, nzflag, pos, (int)nrows, s), "scan");
        int32_t last[2] = {0, 0};
        check(cudaMemcpyAsync(&last[0], pos + nrows - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "D2H");
        check(cudaMemcpyAsync(&last[1], nzflag + nrows - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "D2H");
        check(cudaStreamSynchronize(s), "sync");
        n_nz = (int64_t)last[0] + last[1];
    }
    op.seg_rows = dev_alloc<int32_t>(op, (size_t)std::max<int64_t>(n_nz, 1));
    op.seg_nempty = nrows - n_nz;
    op.seg_empty = dev_alloc<int32_t>(op, (size_t)std::max<int64_t>(op.seg_nempty, 1));
    if (nrows > 0) k_seg_rows<<<grid_for(nrows, 256), 256, 0, s>>>(nrows, nzflag, pos, op.seg_rows, op.seg_empty);
    op.seg_nchunks = nchunks;
    op.seg_cstart = dev_alloc<int32_t>(op, (size_t)nchunks);
    cnt = reinterpret_cast<decltype(cnt)>(analysis_alloc(nchunks * sizeof(int32_t)));
    k_seg_chunkpop<<<grid_for(nchunks, 256), 256, 0, s>>>(nchunks, nwords, op.seg_bits, cnt);
    check(cub::DeviceScan::ExclusiveSum(tmp, tb2, cnt, op.seg_cstart, (int)nchunks, s), "scan");
    // persistent grid: 3 CTAs of 8 warps per SM, a contiguous run of chunks per warp
    int dev = 0, nsm = 148, bps = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_spmv_seg, kSegThreads, 0);
    const int64_t warps = (int64_t)nsm * std::max(1, bps) * (kSegThreads / 32);
    op.seg_cpw = (int)std::max<int64_t>(1, (nchunks + warps - 1) / warps);
    op.seg_nranges = (int)((nchunks + op.seg_cpw - 1) / op.seg_cpw);
    op.seg_grid = (op.seg_nranges + kSegThreads / 32 - 1) / (kSegThreads / 32);
    op.seg_head = dev_alloc<double>(op, (size_t)op.seg_nranges);
    op.seg_tail = dev_alloc<double>(op, (size_t)op.seg_nranges);
    op.seg_flag = dev_alloc<unsigned int>(op, (size_t)op.seg_nranges);
    check(cudaMemsetAsync(op.seg_flag, 0, op.seg_nranges * sizeof(unsigned int), s), "memset");

    check(cudaStreamSynchronize(s), "sync");
    analysis_free(tmp);
    analysis_free(cnt);
    analysis_free(pos);
    analysis_free(nzflag);
    op.seg = true;
}
}  // namespace

void csr_analyze(CsrOp &op, cudaStream_t s) {
    unsigned long long *cnt = dev_alloc<unsigned long long>(op, 16);
    check(cudaMemsetAsync(cnt, 0, 16 * sizeof(unsigned long long), s), "memset");
    k_bin_count<<<grid_for(op.nrows, 256), 256, 0, s>>>(op.nrows, op.row_ptr, cnt);
    unsigned long long hc[9];
    check(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    const unsigned long long max_len = hc[8];
    int64_t off[9];
    off[0] = 0;
    for (int b = 0; b < 8; b++) off[b + 1] = off[b] + (int64_t)hc[b];
    for (int b = 0; b < 8; b++) op.bin_off[b] = off[b];
    op.bin_rows = dev_alloc<int32_t>(op, (size_t)op.nrows);
    {
        uint8_t *k_in = nullptr, *k_out = nullptr;
        int32_t *ids = nullptr;
        void *tmp = nullptr;
        size_t tmp_bytes = 0;
        const int n32 = (int)op.nrows;
        check(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, ids, op.bin_rows, n32, 0, 3, s),
              "radix sort size");
        k_in = reinterpret_cast<decltype(k_in)>(analysis_alloc(std::max<int64_t>(op.nrows, 1) * 2));
        k_out = k_in + std::max<int64_t>(op.nrows, 1);
        ids = reinterpret_cast<decltype(ids)>(analysis_alloc(std::max<int64_t>(op.nrows, 1) * sizeof(int32_t)));
        tmp = reinterpret_cast<decltype(tmp)>(analysis_alloc(std::max<size_t>(tmp_bytes, 1)));
        k_bin_keys<<<grid_for(op.nrows, 256), 256, 0, s>>>(op.nrows, op.row_ptr, k_in, ids);
        check(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, ids, op.bin_rows, n32, 0, 3, s),
              "radix sort");
        check(cudaStreamSynchronize(s), "sync");
        analysis_free(tmp);
        analysis_free(ids);
        analysis_free(k_in);
    }
    // a bin that holds every row lists them in order: the kernels index rows directly
    for (int b = 0; b < 8; b++) op.bin_identity[b] = (off[b + 1] - off[b] == op.nrows);
    // long rows: host-side deterministic chunk table (few rows)
    op.n_long = off[7] - off[6];
    if (op.n_long > 0) {
        std::vector<int32_t> lr(op.n_long);
        std::vector<int64_t> len(op.n_long);
        int64_t *dlen = reinterpret_cast<int64_t *>(analysis_alloc(op.n_long * sizeof(int64_t)));
        k_row_len<<<grid_for(op.n_long, 256), 256, 0, s>>>(op.n_long, op.bin_rows + off[6], op.row_ptr, dlen);
        check(cudaMemcpyAsync(lr.data(), op.bin_rows + off[6], op.n_long * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s), "D2H");
        check(cudaMemcpyAsync(len.data(), dlen, op.n_long * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
        check(cudaStreamSynchronize(s), "sync");
        analysis_free(dlen);
        {  // rows ascending (the bin lists them by key only), lengths alongside
            std::vector<std::pair<int32_t, int64_t>> rl(op.n_long);
            for (int64_t i = 0; i < op.n_long; i++) rl[i] = {lr[i], len[i]};
            std::sort(rl.begin(), rl.end());
            for (int64_t i = 0; i < op.n_long; i++) {
                lr[i] = rl[i].first;
                len[i] = rl[i].second;
            }
        }
        std::vector<int64_t> first(op.n_long + 1);
        std::vector<int32_t> crow;
        int64_t nch = 0;
        for (int64_t i = 0; i < op.n_long; i++) {
            const int64_t L = len[i];
            first[i] = nch;
            int64_t c = (L + kLongRow - 1) / kLongRow;
            for (int64_t q = 0; q < c; q++) crow.push_back((int32_t)i);
            nch += c;
        }
        first[op.n_long] = nch;
        op.n_chunks = nch;
        op.long_rows = dev_alloc<int32_t>(op, op.n_long);
        op.chunk_first = dev_alloc<int64_t>(op, op.n_long + 1);
        op.chunk_row = dev_alloc<int32_t>(op, nch);
        op.chunk_partial = dev_alloc<double>(op, nch);
        check(cudaMemcpyAsync(op.long_rows, lr.data(), op.n_long * sizeof(int32_t), cudaMemcpyHostToDevice, s), "H2D");
        check(cudaMemcpyAsync(op.chunk_first, first.data(), (op.n_long + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s), "H2D");
        check(cudaMemcpyAsync(op.chunk_row, crow.data(), nch * sizeof(int32_t), cudaMemcpyHostToDevice, s), "H2D");
    }
    // schedule choice (SVDSC_POLICY_SPMV 0 = automatic): the row-length bins for
    // small operands and for near-uniform rows of >= 48 nonzeros (measured faster
    // there: config 3 A and A^T 53 vs 60 us, banded config-5 A^T), else the
    // register-segmented chunks (power-law rows, short rows: config 4 A v 696 vs
    // 856 us (round 1's nnz tiles), A^T u 631 vs 758 us (bins))
    bool want_seg = g_policy.spmv == 2;
    if (g_policy.spmv == 0) {
        const double mean = op.nrows > 0 ? (double)op.nnz / (double)op.nrows : 0.0;
        const bool uniform = mean >= 48.0 && (double)max_len <= 1.55 * mean;
        want_seg = op.nnz >= (1 << 20) && !uniform;
    }
    if (want_seg && op.nnz < (int64_t)INT32_MAX &&
        ((reinterpret_cast<uintptr_t>(op.col) & 15) == 0) && ((reinterpret_cast<uintptr_t>(op.val) & 15) == 0))
        seg_analyze(op, s);
    check(cudaStreamSynchronize(s), "sync");
    check(cudaGetLastError(), "analyze");
}

void csr_transpose(const CsrOp &a, CsrOp &at, cudaStream_t s) {
    const int64_t n = a.ncols, nnz = a.nnz;
    at.nrows = n;
    at.ncols = a.nrows;
    at.nnz = nnz;
    int32_t *cnt = dev_alloc<int32_t>(at, (size_t)n);
    int64_t *tp = dev_alloc<int64_t>(at, (size_t)n + 1);
    int32_t *tcol = dev_alloc<int32_t>(at, (size_t)nnz);
    double *tval = dev_alloc<double>(at, (size_t)nnz);
    check(cudaMemsetAsync(cnt, 0, n * sizeof(int32_t), s), "memset");
    k_col_count<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, a.col, cnt);
    // exclusive scan -> tp[0..n-1], tp[n] = nnz
    const int64_t nb = (n + 1023) / 1024;
    int64_t *bsum = nullptr, *boff = nullptr;
    bsum = reinterpret_cast<decltype(bsum)>(analysis_alloc(std::max<int64_t>(nb, 1) * sizeof(int64_t)));
    boff = reinterpret_cast<decltype(boff)>(analysis_alloc(std::max<int64_t>(nb, 1) * sizeof(int64_t)));
    k_scan_block<<<(unsigned)nb, 1024, 0, s>>>(n, cnt, tp, bsum);
    std::vector<int64_t> hb(nb), ho(nb);
    check(cudaMemcpyAsync(hb.data(), bsum, nb * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    int64_t acc = 0;
    for (int64_t i = 0; i < nb; i++) { ho[i] = acc; acc += hb[i]; }
    check(cudaMemcpyAsync(boff, ho.data(), nb * sizeof(int64_t), cudaMemcpyHostToDevice, s), "H2D");
    k_scan_add<<<(unsigned)nb, 1024, 0, s>>>(n, tp, boff);
    check(cudaMemcpyAsync(tp + n, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, s), "H2D");
    // fill keys
    unsigned long long *cursor = nullptr;
    uint64_t *key = nullptr, *tmp = nullptr;
    cursor = reinterpret_cast<decltype(cursor)>(analysis_alloc(std::max<int64_t>(n, 1) * sizeof(unsigned long long)));
    key = reinterpret_cast<decltype(key)>(analysis_alloc(std::max<int64_t>(nnz, 1) * sizeof(uint64_t)));
    static_assert(sizeof(unsigned long long) == sizeof(int64_t), "");
    check(cudaMemcpyAsync(cursor, tp, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s), "D2D");
    k_csc_fill<<<grid_for(a.nrows * 32, 256), 256, 0, s>>>(a.nrows, a.row_ptr, a.col, cursor, key);
    k_seg_sort<<<148 * 8, 256, 0, s>>>(n, tp, key);
    // long columns (> kSegSmem): chunk sort + rank merges (host driven, rare)
    std::vector<int64_t> htp(n + 1);
    check(cudaMemcpyAsync(htp.data(), tp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    for (int64_t c = 0; c < n; c++) {
        int64_t len = htp[c + 1] - htp[c];
        if (len <= kSegSmem) continue;
        if (!tmp) tmp = reinterpret_cast<decltype(tmp)>(analysis_alloc(nnz * sizeof(uint64_t)));
        uint64_t *seg = key + htp[c], *alt = tmp + htp[c];
        k_chunk_sort<<<(unsigned)((len + kSegSmem - 1) / kSegSmem), 256, 0, s>>>(seg, len);
        for (int64_t w = kSegSmem; w < len; w <<= 1) {
            k_merge_runs<<<grid_for(len, 256), 256, 0, s>>>(seg, alt, len, w);
            std::swap(seg, alt);
        }
        if (seg != key + htp[c])
            check(cudaMemcpyAsync(key + htp[c], seg, len * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s), "D2D");
    }
    k_csc_gather<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, key, a.row_ptr, a.val, tcol, tval);
    check(cudaStreamSynchronize(s), "sync");
    check(cudaGetLastError(), "transpose");
    analysis_free(bsum);
    analysis_free(boff);
    analysis_free(cursor);
    analysis_free(key);
    if (tmp) analysis_free(tmp);
    at.row_ptr = tp;
    at.col = tcol;
    at.val = tval;
    csr_analyze(at, s);
}

void spmv_csr(const CsrOp &A, const double *x, double *y, const double *c_dev, const double *yprev,
              const int *abort, cudaStream_t s) {
    if (A.seg) {
        SegArgs sa{A.nnz, (int)A.seg_nchunks, A.seg_cpw, A.seg_nranges, A.col, A.val, x, A.seg_bits,
                   A.seg_rows, A.seg_cstart, A.seg_empty, A.seg_nempty, y, c_dev, yprev, A.seg_head,
                   A.seg_tail, A.seg_flag, abort};
        (void)launch_pdl(k_spmv_seg, dim3(A.seg_grid), dim3(kSegThreads), 0, s, 0, sa);  // errors: cudaGetLastError
        count_launch();
        return;
    }
    const int64_t *o = A.bin_off;
    const int cap = 148 * 8;
    {
        // CTAs per bin proportional to its nonzeros (and rows), >= 1 per non-empty bin
        BinArgs ba{};
        double work[5], tot = 0.0;
        for (int b = 0; b < 5; b++) {
            const int64_t cnt = o[b + 1] - o[b];
            ba.rows[b] = A.bin_identity[b] ? nullptr : A.bin_rows + o[b];
            ba.count[b] = cnt;
            work[b] = cnt > 0 ? (double)cnt * (double)(4 << b) : 0.0;  // rows x typical length class
            tot += work[b];
        }
        static int wave = 0;
        if (!wave) {
            int bps = 0, dev = 0, nsm = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_spmv_bins, 256, 0);
            wave = std::max(1, bps) * nsm;
        }
        const int vcap = std::min(cap, wave);
        int nb_tot = 0;
        for (int b = 0; b < 5; b++) {
            ba.bstart[b] = nb_tot;
            if (ba.count[b] == 0) continue;
            const int G = b == 3 ? kBin3G : (b == 4 ? kBin4G : (2 << b));
            const int need = grid_for(ba.count[b] * G, 256, vcap);
            const int share = std::max(1, (int)(vcap * work[b] / tot + 0.5));
            nb_tot += std::min(need, share);
        }
        ba.bstart[5] = nb_tot;
        if (nb_tot > 0) {
            // one full wave: the grid-stride loops then have no partial second wave
            (void)launch_pdl(k_spmv_bins, dim3(nb_tot), dim3(256), 0, s, 0, ba, (const int64_t *)A.row_ptr,
                             (const int32_t *)A.col, (const double *)A.val, x, y, c_dev, yprev, abort);
            count_launch();
        }
    }
    if (o[6] > o[5]) {
        int64_t cnt = o[6] - o[5];
        k_spmv_cta<<<(unsigned)std::min<int64_t>(cnt, cap), 256, 0, s>>>(A.bin_rows + o[5], cnt, A.row_ptr, A.col,
                                                                          A.val, x, y, c_dev, yprev, abort);
        count_launch();
    }
    if (A.n_long > 0) {
        k_spmv_chunks<<<(unsigned)std::min<int64_t>(A.n_chunks, cap), 256, 0, s>>>(
            A.n_chunks, A.chunk_row, A.chunk_first, A.long_rows, A.row_ptr, A.col, A.val, x, A.chunk_partial, abort);
        k_spmv_chunks_fix<<<grid_for(A.n_long, 128), 128, 0, s>>>(A.n_long, A.long_rows, A.chunk_first,
                                                                  A.chunk_partial, y, c_dev, yprev, abort);
        count_launch();
        count_launch();
    }
}

// ---------------------------------------------------------------------------
// dense GEMV
namespace {

// y_partial[split][r] = sum over this split's columns of A[r, c] x[c]
// CTA = 8 warps over a 64-row strip; warp w takes columns c0 + w + 8q.
template <bool VEC>
__global__ void __launch_bounds__(256) k_gemv_n(int64_t m, int64_t n, const double *__restrict__ A, int64_t ld,
                                                const double *__restrict__ x, double *partial, int64_t cols_per_split,
                                                const int *abort) {
    if (aborted(abort)) return;
    __shared__ double red[8][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r0 = blockIdx.x * 64ll;
    const int64_t c0 = blockIdx.y * cols_per_split;
    const int64_t c1 = min(n, c0 + cols_per_split);
    const int64_t r = r0 + 2 * lane;
    double a0 = 0.0, a1 = 0.0;
    if (VEC && r + 1 < m) {
        const double *base = A + r;
        int64_t c = c0 + w;
        for (; c + 8 * 7 < c1; c += 8 * 8) {
            double2 v[8];
            double xv[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                v[u] = __ldcs(reinterpret_cast<const double2 *>(base + (c + 8 * u) * ld));
                xv[u] = __ldg(x + c + 8 * u);
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                a0 = fma(v[u].x, xv[u], a0);
                a1 = fma(v[u].y, xv[u], a1);
            }
        }
        for (; c < c1; c += 8) {
            double2 v = __ldcs(reinterpret_cast<const double2 *>(base + c * ld));
            double xv = __ldg(x + c);
            a0 = fma(v.x, xv, a0);
            a1 = fma(v.y, xv, a1);
        }
    } else {
        for (int64_t c = c0 + w; c < c1; c += 8) {
            double xv = __ldg(x + c);
            if (r < m) a0 = fma(A[r + c * ld], xv, a0);
            if (r + 1 < m) a1 = fma(A[r + 1 + c * ld], xv, a1);
        }
    }
    red[w][2 * lane] = a0;
    red[w][2 * lane + 1] = a1;
    __syncthreads();
    if (threadIdx.x < 64) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; q++) s += red[q][threadIdx.x];
        const int64_t rr = r0 + threadIdx.x;
        if (rr < m) partial[blockIdx.y * m + rr] = s;
    }
}

// y_partial[split][c] = sum over rows of split of A[r,c] x[r]; warp per column.
template <bool VEC>
__global__ void __launch_bounds__(256) k_gemv_t(int64_t m, int64_t n, const double *__restrict__ A, int64_t ld,
                                                const double *__restrict__ x, double *partial, int64_t rows_per_split,
                                                const int *abort) {
    if (aborted(abort)) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t c = blockIdx.x * 8ll + w;
    const int64_t r0 = blockIdx.y * rows_per_split;
    const int64_t r1 = min(m, r0 + rows_per_split);
    if (c >= n) return;
    const double *col = A + c * ld;
    double acc0 = 0.0, acc1 = 0.0;
    if (VEC) {
        int64_t r = r0 + 2 * lane;
        for (; r + 64 * 7 + 1 < r1; r += 64 * 8) {
            double2 v[8], xv[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                v[u] = __ldcs(reinterpret_cast<const double2 *>(col + r + 64 * u));
                xv[u] = __ldg(reinterpret_cast<const double2 *>(x + r + 64 * u));
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                acc0 = fma(v[u].x, xv[u].x, acc0);
                acc1 = fma(v[u].y, xv[u].y, acc1);
            }
        }
        for (; r + 1 < r1; r += 64) {
            double2 v = __ldcs(reinterpret_cast<const double2 *>(col + r));
            double2 xv = __ldg(reinterpret_cast<const double2 *>(x + r));
            acc0 = fma(v.x, xv.x, acc0);
            acc1 = fma(v.y, xv.y, acc1);
        }
        if (r < r1) acc0 = fma(col[r], x[r], acc0);
    } else {
        for (int64_t r = r0 + lane; r < r1; r += 32) acc0 = fma(col[r], x[r], acc0);
    }
    double s = acc0 + acc1;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) partial[blockIdx.y * n + c] = s;
}

__global__ void k_split_reduce(int64_t len, int splits, const double *__restrict__ partial, double *y,
                               const double *c_dev, const double *yprev, const int *abort) {
    if (aborted(abort)) return;
    const double c = c_dev ? *c_dev : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < splits; q++) s += partial[q * len + i];
        epilogue_store(y, i, s, c, yprev);
    }
}

}  // namespace

void split_reduce(int64_t N, const PreReduce &pr, double *y, const int *abort, cudaStream_t s) {
    k_split_reduce<<<grid_for(N, 256), 256, 0, s>>>(N, pr.splits, pr.partial, y, pr.c_dev, pr.yprev, abort);
    count_launch();
}

void gemv_n(const DenseOp &A, const double *x, double *y, const double *c_dev, const double *yprev,
            const int *abort, cudaStream_t s) {
    const int64_t m = A.nrows, n = A.ncols;
    const int64_t rb = (m + 63) / 64;
    const int splits = A.splits_n;
    const int64_t cps = (n + splits - 1) / splits;
    dim3 grid((unsigned)rb, (unsigned)splits);
    const bool vec = (A.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(A.data) & 15) == 0);
    if (vec) k_gemv_n<true><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, cps, abort);
    else k_gemv_n<false><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, cps, abort);
    k_split_reduce<<<grid_for(m, 256), 256, 0, s>>>(m, splits, A.partial, y, c_dev, yprev, abort);
    count_launch();
    count_launch();
}

void gemv_t(const DenseOp &A, const double *x, double *y, const double *c_dev, const double *yprev,
            const int *abort, cudaStream_t s) {
    const int64_t m = A.nrows, n = A.ncols;
    const int splits = A.splits_t;
    int64_t rps = (m + splits - 1) / splits;
    rps = (rps + 1) & ~1ll;  // even, keeps 16-byte alignment of every split start
    const bool vec = (A.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(A.data) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    {
        dim3 grid((unsigned)((n + 7) / 8), (unsigned)splits);
        if (vec) k_gemv_t<true><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, rps, abort);
        else k_gemv_t<false><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, rps, abort);
    }
    k_split_reduce<<<grid_for(n, 256), 256, 0, s>>>(n, splits, A.partial, y, c_dev, yprev, abort);
    count_launch();
    count_launch();
}

// the products without their split-K reduction (finished by the next CGS2 kernel)
void gemv_n_partial(const DenseOp &A, const double *x, PreReduce &pr, const double *c_dev, const double *yprev,
                    const int *abort, cudaStream_t s) {
    const int64_t m = A.nrows, n = A.ncols;
    const int64_t rb = (m + 63) / 64;
    const int splits = A.splits_n;
    const int64_t cps = (n + splits - 1) / splits;
    dim3 grid((unsigned)rb, (unsigned)splits);
    const bool vec = (A.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(A.data) & 15) == 0);
    if (vec) k_gemv_n<true><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, cps, abort);
    else k_gemv_n<false><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, cps, abort);
    count_launch();
    pr.partial = A.partial;
    pr.splits = splits;
    pr.c_dev = c_dev;
    pr.yprev = yprev;
}

void gemv_t_partial(const DenseOp &A, const double *x, PreReduce &pr, const double *c_dev, const double *yprev,
                    const int *abort, cudaStream_t s) {
    const int64_t m = A.nrows, n = A.ncols;
    const int splits = A.splits_t;
    int64_t rps = (m + splits - 1) / splits;
    rps = (rps + 1) & ~1ll;
    const bool vec = (A.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(A.data) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    dim3 grid((unsigned)((n + 7) / 8), (unsigned)splits);
    if (vec) k_gemv_t<true><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, rps, abort);
    else k_gemv_t<false><<<grid, 256, 0, s>>>(m, n, A.data, A.ld, x, A.partial, rps, abort);
    count_launch();
    pr.partial = A.partial;
    pr.splits = splits;
    pr.c_dev = c_dev;
    pr.yprev = yprev;
}

// ---------------------------------------------------------------------------
// Column split of a rank's rows (multi-GPU A v): loc holds the
// entries whose column lies in [c0, c1) (the rank's own slice of v, columns
// rebased to c - c0), rem the others (global columns), each row's entries in
// their original order.  A v = loc v_slice + rem v_full: the first product
// runs while the all-gather of v is in flight.
namespace {
__global__ void k_split_count(int64_t nrows, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                              int32_t c0, int32_t c1, int64_t *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < nrows; r += nw) {
        int64_t c = 0;
        for (int64_t p = rp[r] + lane; p < rp[r + 1]; p += 32) c += (col[p] >= c0 && col[p] < c1);
        for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
        if (lane == 0) cnt[r] = c;
    }
}
__global__ void k_split_fill(int64_t nrows, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                             const double *__restrict__ val, int32_t c0, int32_t c1, const int64_t *__restrict__ rpl,
                             int32_t *__restrict__ coll, double *__restrict__ vall, int64_t *__restrict__ rpr,
                             int32_t *__restrict__ colr, double *__restrict__ valr) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r <= nrows; r += nw) {
        if (r == nrows) {  // last row pointer of rem
            if (lane == 0) rpr[nrows] = rp[nrows] - rpl[nrows];
            continue;
        }
        int64_t ol = rpl[r], orm = rp[r] - rpl[r];
        if (lane == 0) rpr[r] = orm;
        for (int64_t p0 = rp[r]; p0 < rp[r + 1]; p0 += 32) {
            const int64_t p = p0 + lane;
            const bool ok = p < rp[r + 1];
            const int32_t c = ok ? col[p] : 0;
            const bool isl = ok && c >= c0 && c < c1;
            const unsigned ml = __ballot_sync(0xffffffffu, isl), mr = __ballot_sync(0xffffffffu, ok && !isl);
            const unsigned below = (1u << lane) - 1u;
            if (isl) {
                coll[ol + __popc(ml & below)] = c - c0;
                vall[ol + __popc(ml & below)] = val[p];
            } else if (ok) {
                colr[orm + __popc(mr & below)] = c;
                valr[orm + __popc(mr & below)] = val[p];
            }
            ol += __popc(ml);
            orm += __popc(mr);
        }
    }
}
}  // namespace

void csr_split_columns(const CsrOp &a, int64_t c0, int64_t c1, CsrOp &loc, CsrOp &rem, cudaStream_t s) {
    const int64_t nrows = a.nrows;
    int64_t *cnt = reinterpret_cast<int64_t *>(analysis_alloc((nrows + 1) * sizeof(int64_t)));
    check(cudaMemsetAsync(cnt, 0, (nrows + 1) * sizeof(int64_t), s), "memset");
    if (nrows > 0)
        k_split_count<<<grid_for(nrows * 32, 256), 256, 0, s>>>(nrows, a.row_ptr, a.col, (int32_t)c0, (int32_t)c1, cnt);
    int64_t *rpl = dev_alloc<int64_t>(loc, (size_t)nrows + 1);
    size_t tb = 0;
    check(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, rpl, (int)(nrows + 1), s), "scan size");
    void *tmp = analysis_alloc(std::max<size_t>(tb, 1));
    check(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, rpl, (int)(nrows + 1), s), "scan");
    int64_t nl = 0;
    check(cudaMemcpyAsync(&nl, rpl + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    analysis_free(tmp);
    analysis_free(cnt);
    const int64_t nr = a.nnz - nl;
    int32_t *coll = dev_alloc<int32_t>(loc, (size_t)std::max<int64_t>(nl, 1));
    double *vall = dev_alloc<double>(loc, (size_t)std::max<int64_t>(nl, 1));
    int64_t *rpr = dev_alloc<int64_t>(rem, (size_t)nrows + 1);
    int32_t *colr = dev_alloc<int32_t>(rem, (size_t)std::max<int64_t>(nr, 1));
    double *valr = dev_alloc<double>(rem, (size_t)std::max<int64_t>(nr, 1));
    k_split_fill<<<grid_for((nrows + 1) * 32, 256), 256, 0, s>>>(nrows, a.row_ptr, a.col, a.val, (int32_t)c0,
                                                                (int32_t)c1, rpl, coll, vall, rpr, colr, valr);
    check(cudaGetLastError(), "k_split_fill");
    loc.nrows = rem.nrows = nrows;
    loc.ncols = c1 - c0;
    rem.ncols = a.ncols;
    loc.nnz = nl;
    rem.nnz = nr;
    loc.row_ptr = rpl;
    loc.col = coll;
    loc.val = vall;
    rem.row_ptr = rpr;
    rem.col = colr;
    rem.val = valr;
    csr_analyze(loc, s);
    csr_analyze(rem, s);
}

// rows [r0, r1) of a CSR operand as a standalone operand (row pointers rebased,
// column / value arrays shared with `a`), analysed for the product kernels
namespace {
__global__ void k_rebase_rows(int64_t n, const int64_t *__restrict__ rp, int64_t base, int64_t *__restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n; r += (int64_t)gridDim.x * blockDim.x)
        out[r] = rp[r] - base;
}
}  // namespace

void csr_row_slice(const CsrOp &a, int64_t r0, int64_t r1, CsrOp &out, cudaStream_t s) {
    int64_t b[2] = {0, 0};
    check(cudaMemcpyAsync(&b[0], a.row_ptr + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaMemcpyAsync(&b[1], a.row_ptr + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    const int64_t n = r1 - r0;
    int64_t *rp = dev_alloc<int64_t>(out, (size_t)n + 1);
    k_rebase_rows<<<grid_for(n + 1, 256), 256, 0, s>>>(n, a.row_ptr + r0, b[0], rp);
    check(cudaGetLastError(), "k_rebase_rows");
    out.nrows = n;
    out.ncols = a.ncols;
    out.nnz = b[1] - b[0];
    out.row_ptr = rp;
    out.col = a.col + b[0];
    out.val = a.val + b[0];
    csr_analyze(out, s);
}

}  // namespace svdsc
