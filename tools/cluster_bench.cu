// Launch / cluster-barrier cost microbenchmark (B200): back-to-back launches
// timed with events (per-launch time = launch throughput incl. gaps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_bench tools/cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_empty(int *p) {
    if (p && threadIdx.x == 9999) *p = 1;
}
__global__ void k_csync(int *p, int n) {
    extern __shared__ double sm[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = 0; i < n; i++) cl.sync();
    if (p && threadIdx.x == 9999) *p = (int)sm[0];
}

template <class F>
float timeit(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 20; i++) f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; i++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return 1000.f * ms / reps;
}

float cl_launch(int C, int thr, size_t smem, int nsync, bool graph) {
    cudaFuncSetAttribute(k_csync, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_csync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(thr);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaStream_t s;
    cudaStreamCreate(&s);
    cfg.stream = s;
    auto f = [&] { cudaLaunchKernelEx(&cfg, k_csync, (int *)nullptr, nsync); };
    float r;
    if (!graph) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int i = 0; i < 20; i++) f();
        cudaEventRecord(a, s);
        for (int i = 0; i < 1000; i++) f();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        r = ms;
    } else {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 100; i++) f();
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int i = 0; i < 10; i++) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        r = ms;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return r;  // ms per 1000 launches = us per launch
}

int main() {
    printf("empty 16x512: %.2f us\n", timeit([] { k_empty<<<16, 512>>>(nullptr); }, 2000));
    printf("empty 148x512: %.2f us\n", timeit([] { k_empty<<<148, 512>>>(nullptr); }, 2000));
    printf("empty 1x128: %.2f us\n", timeit([] { k_empty<<<1, 128>>>(nullptr); }, 2000));
    for (bool gr : {false, true})
        for (int C : {8, 16})
            for (size_t sm : {(size_t)0, (size_t)80 * 1024, (size_t)190 * 1024})
                for (int ns : {0, 1, 10}) {
                    printf("%s cluster C=%d smem=%zuK sync=%d: %.2f us/launch\n", gr ? "graph" : "stream", C, sm / 1024,
                           ns, cl_launch(C, 512, sm, ns, gr));
                }
    return 0;
}
