// Microbenchmark: latency of one cluster-wide barrier on B200 for the
// variants the march kernel could use.  Not part of the product.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void bar_kernel(int iters, long long *out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
            cg::this_cluster().sync();
        } else if (MODE == 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else if (MODE == 2) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        } else {
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}

template <int MODE>
float run(int cs, int threads, int iters) {
    long long *d;
    cudaMalloc(&d, 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cs > 8) cudaFuncSetAttribute(bar_kernel<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, bar_kernel<MODE>, iters, d);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, bar_kernel<MODE>, iters, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    printf("mode=%d cs=%2d threads=%4d : %7.1f ns/barrier (%lld cycles)  err=%s\n", MODE, cs, threads,
           ms * 1e6 / iters, cyc, cudaGetErrorString(cudaGetLastError()));
    return ms;
}

int main() {
    const int iters = 20000;
    for (int cs : {2, 4, 8, 16})
        for (int t : {128, 256}) {
            run<0>(cs, t, iters);
            run<1>(cs, t, iters);
            run<2>(cs, t, iters);
        }
    run<3>(1, 128, iters);
    run<3>(1, 512, iters);
    return 0;
}
