// barrier_bench.cu -- cost of a grid-wide barrier on B200 (profiling aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/barrier_bench.cu && /tmp/bb
// Variants, each a cooperative launch of G CTAs doing R barriers:
//   0  arrival atomicAdd (returning) + last-arriver generation bump (cgs_fused.cu grid_sync)
//   1  monotonic counter: red.release.gpu.add + ld.acquire poll until >= target
//   2  variant 1 inside thread-block clusters of 8: barrier.cluster, then one CTA
//      per cluster arrives globally, then barrier.cluster again
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_bar0(unsigned *flags, int R) {
    for (int r = 0; r < R; r++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned gen = ld_acq(flags + 1);
            __threadfence();
            if (atomicAdd(flags, 1u) == gridDim.x - 1) {
                flags[0] = 0;
                __threadfence();
                atomicAdd(flags + 1, 1u);
            } else {
                while (ld_acq(flags + 1) == gen) __nanosleep(20);
            }
            __threadfence();
        }
        __syncthreads();
    }
}

__global__ void k_bar1(unsigned *flags, int R) {
    for (int r = 1; r <= R; r++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            red_rel(flags, 1u);
            const unsigned target = (unsigned)r * gridDim.x;
            while (ld_acq(flags) < target) {
            }
        }
        __syncthreads();
    }
}

__global__ void k_bar2(unsigned *flags, int R) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned ncl = gridDim.x / cl.num_blocks();
    for (int r = 1; r <= R; r++) {
        cl.sync();
        if (cl.block_rank() == 0 && threadIdx.x == 0) {
            red_rel(flags, 1u);
            const unsigned target = (unsigned)r * ncl;
            while (ld_acq(flags) < target) {
            }
        }
        cl.sync();
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned *flags;
    cudaMalloc(&flags, 64);
    const int R = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int per_sm = 1; per_sm <= 2; per_sm++) {
        const int G = nsm * per_sm;
        for (int v = 0; v < 3; v++) {
            if (v == 2 && G % 8) continue;
            float best = 1e30f;
            for (int rep = 0; rep < 3; rep++) {
                cudaMemset(flags, 0, 64);
                int Rr = R;
                void *args[] = {&flags, &Rr};
                cudaEventRecord(e0);
                if (v == 0) cudaLaunchCooperativeKernel((void *)k_bar0, G, 256, args, 0, 0);
                if (v == 1) cudaLaunchCooperativeKernel((void *)k_bar1, G, 256, args, 0, 0);
                if (v == 2) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(G);
                    cfg.blockDim = dim3(256);
                    cudaLaunchAttribute at[2];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = 8;
                    at[0].val.clusterDim.y = 1;
                    at[0].val.clusterDim.z = 1;
                    at[1].id = cudaLaunchAttributeCooperative;
                    at[1].val.cooperative = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 2;
                    cudaLaunchKernelEx(&cfg, k_bar2, flags, Rr);
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            cudaError_t err = cudaGetLastError();
            printf("G=%d variant=%d  %.3f us per barrier  %s\n", G, v, best * 1e3f / R,
                   err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
    }
    return 0;
}
