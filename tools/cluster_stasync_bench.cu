// Microbenchmark: all-to-all exchange of one double per CTA through
// st.async + mbarrier complete_tx (no cluster barrier), vs the hardware
// cluster barrier.  Not part of the product.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

template <int CS>
__global__ void xchg_kernel(int iters, long long *out, double *res) {
    __shared__ alignas(8) unsigned long long mbar[2];
    __shared__ alignas(8) double slot[2][16];
    const int q = blockIdx.x % CS;
    if (threadIdx.x == 0) {
        for (int p = 0; p < 2; ++p)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar[p])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int p = i & 1;
        const unsigned phase = (i >> 1) & 1;
        if (threadIdx.x == 0) {
            // expect CS * 8 bytes this phase
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         ::"r"(smem_u32(&mbar[p])), "r"(CS * 8) : "memory");
        }
        if (threadIdx.x < CS) {
            const int j = threadIdx.x;
            unsigned raddr, rbar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(&slot[p][q])), "r"(j));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&mbar[p])), "r"(j));
            const double v = (double)(q + i);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                         ::"r"(raddr), "d"(v), "r"(rbar) : "memory");
        }
        unsigned done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&mbar[p])), "r"(phase) : "memory");
        }
        double m = slot[p][0];
        for (int j = 1; j < CS; ++j) m = m > slot[p][j] ? m : slot[p][j];
        acc += m;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
    if (threadIdx.x == 0) res[blockIdx.x] = acc;
    cg::this_cluster().sync();
}

template <int CS>
void run(int threads, int iters) {
    long long *d; double *r;
    cudaMalloc(&d, 8); cudaMalloc(&r, 8 * 64);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    if (CS > 8) cudaFuncSetAttribute(xchg_kernel<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchKernelEx(&cfg, xchg_kernel<CS>, iters, d, r);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, xchg_kernel<CS>, iters, d, r);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    double h[64]; cudaMemcpy(h, r, 8 * CS, cudaMemcpyDeviceToHost);
    printf("st.async all-to-all cs=%2d threads=%d: %7.1f ns/exchange (%lld cycles) check=%g err=%s\n",
           CS, threads, ms * 1e6 / iters, cyc, h[0], cudaGetErrorString(cudaGetLastError()));
    cudaFree(d); cudaFree(r);
}

int main() {
    run<2>(128, 20000);
    run<4>(128, 20000);
    run<8>(128, 20000);
    run<16>(128, 20000);
    return 0;
}
