// Dependent-latency microbenchmark (cycles per op, one warp): DFMA, DADD, FFMA,
// MUFU rcp/rsqrt f64 approx, SHFL (64-bit value), bar.sync with 4 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double *out, long long *cyc, double x0, float f0) {
    const int N = 1024;
    double x = x0 + threadIdx.x * 1e-20;
    float f = f0;
    long long t0, t1;
    __syncthreads();
    // DFMA chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = fma(x, 0.999999, 1e-9);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x + 1e-9;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // FFMA chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) f = fmaf(f, 0.9999f, 1e-6f);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // rcp.approx.ftz.f64 chain
    double y = x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(y));
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // rsqrt.approx.f64 chain (of |y|+1)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) asm volatile("rsqrt.approx.f64 %0, %0;" : "+d"(y));
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // SHFL of a double + DADD
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x += __shfl_xor_sync(0xffffffffu, x, 1);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = t1 - t0;
    // bar.sync
    t0 = clock64();
    for (int i = 0; i < N; i++) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = t1 - t0;
    // sqrt (IEEE f64)
    t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N; i++) y = sqrt(y + 1.0);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[7] = t1 - t0;
    // DMUL chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x * 1.0000001;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[8] = t1 - t0;
    // DSETP + select chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = (x > 1.0) ? x * 0.5 : x + 0.25;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[9] = t1 - t0;
    out[threadIdx.x] = x + y + f;
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMallocManaged(&cyc, 16 * 8);
    const char *names[] = {"DFMA", "DADD", "FFMA", "rcp.approx.f64", "rsqrt.approx.f64", "SHFL64+DADD",
                           "bar.sync", "sqrt+1 f64", "DMUL", "DSETP+sel"};
    for (int warps : {1, 4, 16}) {
        k<<<1, 32 * warps>>>(out, cyc, 1.5, 1.5f);
        k<<<1, 32 * warps>>>(out, cyc, 1.5, 1.5f);
        cudaDeviceSynchronize();
        printf("warps=%d:", warps);
        for (int i = 0; i < 10; i++) printf(" %s=%.1f", names[i], cyc[i] / 1024.0);
        printf("\n");
    }
    return 0;
}
