// Microbenchmark: HBM read bandwidth of TMA row-tile streaming of a tall
// column-major N x C basis (ld = N), the access pattern of the CGS2 kernel.
// One CTA per SM owns a contiguous row range; one producer thread issues
// boxes of BR rows x 16 columns into NS stages of BR rows x CC columns
// (full/empty mbarriers); 16 consumer warps touch each stage and release it.
// Also: a contiguous bulk-copy reference (row-panel layout).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tb tools/tma_bw.cu -lcuda && /tmp/tb 200000 300
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, unsigned ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     su(b)),
                 "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, int c0, int c1, uint64_t *b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su(dst)),
        "l"(m), "r"(c0), "r"(c1), "r"(su(b))
        : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, unsigned bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)),
                 "l"(src), "r"(bytes), "r"(su(b))
                 : "memory");
}

// mode 0: TMA boxes BR x 16 of a column-major matrix; stage = BR rows x CC cols
// mode 1: contiguous bulk copies of `chunk` bytes (row-panel layout reference)
__global__ void __launch_bounds__(544, 1) k_stream(const __grid_constant__ CUtensorMap tm, const double *Q, int64_t N, int C,
                                                   int BR, int CC, int NS, int mode, int64_t chunk, double *sink) {
    extern __shared__ __align__(1024) double sm[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    const int64_t rpb = ((N + gridDim.x - 1) / gridDim.x + BR - 1) / BR * BR;
    const int64_t rb = blockIdx.x * rpb, re = rb + rpb < N ? rb + rpb : N;
    const int nrt = rb < re ? (int)((re - rb + BR - 1) / BR) : 0;
    const int ncc = (C + CC - 1) / CC;
    const int nunits = mode == 0 ? nrt * ncc : (int)(((re - rb) * C * 8 + chunk - 1) / chunk);
    const int stage_d = mode == 0 ? BR * CC : (int)(chunk / 8);
    if (tid == 0) {
        for (int q = 0; q < NS; q++) mb_init(&full[q], 1), mb_init(&empty[q], 16);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc = 0.0;
    if (wid == 16) {
        if (lane == 0)
            for (int u = 0; u < nunits; u++) {
                const int st = u % NS;
                if (u >= NS) mb_wait(&empty[st], ((u / NS) - 1) & 1);
                double *dst = sm + (size_t)st * stage_d;
                if (mode == 0) {
                    const int rt = u / ncc, cc = u % ncc;
                    const int c0 = cc * CC, nc = C - c0 < CC ? C - c0 : CC;
                    const int nb = (nc + 15) / 16;
                    mb_tx(&full[st], (unsigned)(nb * BR * 16 * 8));
                    for (int b = 0; b < nb; b++) tma2d(dst + b * BR * 16, &tm, (int)(rb + (int64_t)rt * BR), c0 + 16 * b, &full[st]);
                } else {
                    const int64_t off = rb * C * 8 + (int64_t)u * chunk;
                    const int64_t end = re * C * 8;
                    const unsigned bytes = (unsigned)(end - off < chunk ? end - off : chunk);
                    mb_tx(&full[st], bytes);
                    bulk(dst, reinterpret_cast<const char *>(Q) + off, bytes, &full[st]);
                }
            }
    } else {
        for (int u = 0; u < nunits; u++) {
            const int st = u % NS;
            mb_wait(&full[st], (u / NS) & 1);
            acc += sm[(size_t)st * stage_d + (tid & 255)];
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[st]);
        }
    }
    if (acc == 123.456) sink[0] = acc;
}

int main(int argc, char **argv) {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int64_t N = argc > 1 ? atoll(argv[1]) : 200000;
    const int C = argc > 2 ? atoi(argv[2]) : 300;
    const int64_t ld = (N + 31) / 32 * 32;
    double *Q, *sink;
    cudaMalloc(&Q, (size_t)ld * C * 8 + 4096);
    cudaMalloc(&sink, 8);
    cudaMemset(Q, 0, (size_t)ld * C * 8);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)N * C * 8;
    printf("N=%lld C=%d\n", (long long)N, C);
    auto run = [&](const char *nm, int BR, int CC, int mode, int64_t chunk) {
        CUtensorMap tm;
        cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)C};
        cuuint64_t gstr[1] = {(cuuint64_t)ld * 8};
        cuuint32_t box[2] = {(cuuint32_t)BR, 16};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Q, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const size_t stage_b = mode == 0 ? (size_t)BR * CC * 8 : (size_t)chunk;
        int NS = (int)((200 * 1024) / stage_b);
        if (NS > 16) NS = 16;
        if (NS < 1) return;
        const size_t smem = NS * stage_b;
        auto launch = [&] { k_stream<<<nsm, 544, smem>>>(tm, Q, N, C, BR, CC, NS, mode, chunk, sink); };
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 5; i++) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s NS=%2d %8.1f GB/s (%s)\n", nm, NS, bytes * 5 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    run("tma BR=16 CC=all", 16, (C + 15) / 16 * 16, 0, 0);
    run("tma BR=32 CC=all", 32, (C + 15) / 16 * 16, 0, 0);
    run("tma BR=64 CC=64", 64, 64, 0, 0);
    run("tma BR=64 CC=128", 64, 128, 0, 0);
    run("tma BR=128 CC=32", 128, 32, 0, 0);
    run("tma BR=128 CC=64", 128, 64, 0, 0);
    run("tma BR=256 CC=16", 256, 16, 0, 0);
    run("tma BR=256 CC=32", 256, 32, 0, 0);
    run("bulk contiguous 16KB", 16, 16, 1, 16384);
    run("bulk contiguous 32KB", 16, 16, 1, 32768);
    return 0;
}
