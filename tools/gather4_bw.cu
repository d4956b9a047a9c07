// Microbenchmark: random 8-byte gathers through the TMA engine
// (cp.async.bulk.tensor.2d ... tile::gather4: four 16-byte rows of x viewed as
// an (n/2) x 2 tensor per instruction, into shared memory, mbarrier
// completion) versus plain LDG gathers (tools/gather_bw.cu "gonly", ~1 gather
// per SM-cycle: the L1 wavefront rate).  Question: can a random-gather SpMV
// leave the L1 t-stage bound by gathering through TMA?
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather4_bw.cu -lcuda -o tools/gather4_bw
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t z) {
    z ^= z >> 16; z *= 0x7feb352dU; z ^= z >> 15; z *= 0x846ca68bU; z ^= z >> 16;
    return z;
}

constexpr int kOpsPerStage = 128;   // gather4 ops per stage per CTA (512 gathered rows)
constexpr int kStages = 4;

__global__ void __launch_bounds__(128) k_gather4(const __grid_constant__ CUtensorMap tm, int64_t ngroups, uint32_t nrows,
                                                 double *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    double *buf = reinterpret_cast<double *>(sm);                   // kStages x kOpsPerStage x 4 rows x 2 doubles
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + kStages * kOpsPerStage * 128);
    const int tid = threadIdx.x;
    if (tid < kStages) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + tid);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // this CTA's groups of kOpsPerStage ops
    const int64_t per = (ngroups + gridDim.x - 1) / gridDim.x;
    const int64_t g0 = blockIdx.x * per, g1 = min(ngroups, g0 + per);
    double acc = 0.0;
    uint32_t phase[kStages] = {0, 0, 0, 0};
    auto issue = [&](int64_t g, int st) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + st);
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kOpsPerStage * 64) : "memory");
        __syncthreads();
        // thread t issues op t of the stage: 4 random rows
        const uint32_t base = (uint32_t)(g * kOpsPerStage + tid) * 4u;
        int32_t r[4];
#pragma unroll
        for (int u = 0; u < 4; u++)
            r[u] = (int32_t)(((uint64_t)hash32((base + u) * 2654435761U + 12345U) * (uint64_t)nrows) >> 32);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + ((size_t)st * kOpsPerStage + tid) * 16);  // 128-B aligned
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            :
            : "r"(dst), "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(b)
            : "memory");
    };
    int64_t gi = g0;
    for (int s = 0; s < kStages && gi < g1; s++, gi++) issue(gi, s);
    int st = 0;
    for (int64_t g = g0; g < g1; g++) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + st);
        uint32_t done = 0;
        long long spins = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(b), "r"(phase[st]) : "memory");
            if (++spins > (1LL << 24)) {  // a malformed copy never completes: bail out
                sink[1] = 1.0;
                return;
            }
        }
        phase[st] ^= 1u;
        const double *v = buf + ((size_t)st * kOpsPerStage + tid) * 16;
        acc += v[0] + v[3] + v[4] + v[7];
        __syncthreads();  // the stage is consumed before it is refilled
        if (gi < g1) issue(gi++, st);
        st = (st + 1) % kStages;
    }
    if (acc == 1.2345e300) sink[0] = acc;
}

int main(int argc, char **argv) {
    const int64_t ngather = argc > 1 ? atoll(argv[1]) : 150000000LL;
    const int64_t n = argc > 2 ? atoll(argv[2]) : 2000000;
    int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    double *x, *sink;
    CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&sink, 16)); CK(cudaMemset(sink, 0, 16));
    CK(cudaMemset(x, 0, n * 8));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    const size_t smem = kStages * kOpsPerStage * 128 + 64;
    CK(cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ngroups = ngather / (4 * kOpsPerStage);
    for (int bps : {1, 2, 4, 8}) {
        const int grid = nsm * bps;
        k_gather4<<<grid, 128, smem>>>(tm, ngroups, (uint32_t)(n / 2), sink);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a));
        for (int r = 0; r < 5; r++) k_gather4<<<grid, 128, smem>>>(tm, ngroups, (uint32_t)(n / 2), sink);
        CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        const double us = ms * 1000.0 / 5;
        const double g = (double)ngroups * 4 * kOpsPerStage;
        printf("{\"kernel\": \"tma_gather4\", \"ctas_per_sm\": %d, \"gathers\": %.0f, \"n\": %lld, \"us\": %.1f, "
               "\"ggather_per_s\": %.2f}\n", bps, g, (long long)n, us, g / (us * 1e3));
    }
    double hs[2];
    CK(cudaMemcpy(hs, sink, 16, cudaMemcpyDeviceToHost));
    if (hs[1] != 0.0) printf("{\"error\": \"a gather4 stage never completed\"}\n");
    CK(cudaGetLastError());
    return 0;
}
