// Microbenchmark: the memory-side ceiling of a CSR SpMV whose column indices
// are uniformly random (BASELINE config 4: 150M nonzeros, x of 2M doubles).
// Every nonzero costs one 4-byte index + one 8-byte value streamed from HBM
// (the algorithmic 12 B) and one random 8-byte gather of x.  The kernels below
// do exactly those memory operations and nothing else a real SpMV needs (no
// row boundaries, no segmented sums), so their rate bounds k_spmv_seg from
// above:
//   stream  : index + value streams only (no gathers)           -> HBM ceiling
//   gather  : streams + one x gather per nonzero (default cache) -> gather ceiling
//   gnc     : same, gathers through ld.global.nc.L1::no_allocate
//   gonly   : gathers with indices generated in registers (no streams)
// Output: one line per kernel with us, nonzeros/s and algorithmic GB/s (12 B
// per nonzero).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//   tools/gather_bw.cu -o tools/gather_bw ; run: tools/gather_bw [nnz] [n]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t z) {
    z ^= z >> 16; z *= 0x7feb352dU; z ^= z >> 15; z *= 0x846ca68bU; z ^= z >> 16;
    return z;
}

__global__ void k_fill(int32_t *col, double *val, int64_t nnz, int32_t n) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
        col[j] = (int32_t)(((uint64_t)hash32((uint32_t)j * 2654435761U + 12345U) * (uint64_t)n) >> 32);
        val[j] = 1.0 + (double)(j & 7);
    }
}

template <int MODE>
__device__ __forceinline__ double gx(const double *x, int32_t c) {
    if (MODE == 2) {
        double v;
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(x + c));
        return v;
    }
    return __ldg(x + c);
}

// MODE 0: streams only, 1: streams + gather, 2: streams + nc/no_allocate gather
template <int MODE>
__global__ void __launch_bounds__(256) k_run(const int32_t *__restrict__ col, const double *__restrict__ val,
                                             const double *__restrict__ x, int64_t nnz, double *sink) {
    const int64_t q = nnz / 4;  // groups of 4 nonzeros per lane per iteration
    double acc = 0.0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < q; g += (int64_t)gridDim.x * blockDim.x) {
        const int4 c = __ldcs(reinterpret_cast<const int4 *>(col) + g);
        const double2 v0 = __ldcs(reinterpret_cast<const double2 *>(val) + 2 * g);
        const double2 v1 = __ldcs(reinterpret_cast<const double2 *>(val) + 2 * g + 1);
        if (MODE == 0) {
            acc += v0.x * c.x + v0.y * c.y + v1.x * c.z + v1.y * c.w;
        } else {
            acc += v0.x * gx<MODE>(x, c.x) + v0.y * gx<MODE>(x, c.y) + v1.x * gx<MODE>(x, c.z) +
                   v1.y * gx<MODE>(x, c.w);
        }
    }
    if (acc == 1.2345e300) sink[0] = acc;
}

__global__ void __launch_bounds__(256) k_gonly(const double *__restrict__ x, int64_t nnz, int32_t n, double *sink) {
    const int64_t q = nnz / 4;
    double acc = 0.0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < q; g += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t h = hash32((uint32_t)(4 * g + u) * 2654435761U + 12345U);
            acc += __ldg(x + (int32_t)(((uint64_t)h * (uint64_t)n) >> 32));
        }
    }
    if (acc == 1.2345e300) sink[0] = acc;
}

template <class F>
static float timeit(F f, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    f(); CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; r++) f();
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    return ms * 1000.f / reps;
}

int main(int argc, char **argv) {
    const int64_t nnz = argc > 1 ? atoll(argv[1]) : 150000000LL;
    const int32_t n = argc > 2 ? atoi(argv[2]) : 2000000;
    int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t *col; double *val, *x, *sink;
    CK(cudaMalloc(&col, nnz * 4)); CK(cudaMalloc(&val, nnz * 8));
    CK(cudaMalloc(&x, (int64_t)n * 8)); CK(cudaMalloc(&sink, 8));
    k_fill<<<nsm * 8, 256>>>(col, val, nnz, n);
    CK(cudaMemset(x, 0, (int64_t)n * 8));
    CK(cudaDeviceSynchronize());
    const double alg = 12.0 * (double)nnz;
    for (int bps : {4, 8}) {
        const int grid = nsm * bps;
        struct { const char *name; float us; } r[4] = {
            {"stream", timeit([&] { k_run<0><<<grid, 256>>>(col, val, x, nnz, sink); }, 10)},
            {"gather", timeit([&] { k_run<1><<<grid, 256>>>(col, val, x, nnz, sink); }, 10)},
            {"gnc", timeit([&] { k_run<2><<<grid, 256>>>(col, val, x, nnz, sink); }, 10)},
            {"gonly", timeit([&] { k_gonly<<<grid, 256>>>(x, nnz, n, sink); }, 10)},
        };
        for (auto &e : r)
            printf("{\"kernel\": \"%s\", \"ctas_per_sm\": %d, \"nnz\": %lld, \"n\": %d, \"us\": %.1f, "
                   "\"gnnz_per_s\": %.2f, \"alg_GBps\": %.0f}\n",
                   e.name, bps, (long long)nnz, n, e.us, nnz / (e.us * 1e3), alg / (e.us * 1e3));
    }
    CK(cudaGetLastError());
    return 0;
}
