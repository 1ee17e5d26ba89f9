// Probe: how many thread-block clusters of a given size / shared-memory
// footprint can be resident at once on this GPU (cudaOccupancyMaxActiveClusters).
// Usage: cluster_occupancy  -> prints one line per (cluster size, smem KB, threads).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(double *p) {
    extern __shared__ double s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (p) p[blockIdx.x] = s[0];
}

int main() {
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int css[] = {1, 2, 4, 8, 16};
    const int kbs[] = {40, 70, 100, 140, 200};
    const int thr[] = {128, 256, 512};
    for (int cs : css)
        for (int kb : kbs)
            for (int nt : thr) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs * 64);
                cfg.blockDim = dim3(nt);
                cfg.dynamicSmemBytes = (size_t)kb * 1024;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = cs;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                int n = -1;
                cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
                printf("sms %d cluster %2d smem_kb %3d threads %3d max_active_clusters %4d ctas %4d %s\n",
                       sms, cs, kb, nt, n, n * cs, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
