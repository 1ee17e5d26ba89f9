// Dependent-chain latency of FP64 operations on B200 (one warp, clock64),
// to size the latency hiding of the propagator kernels.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double *out, long long *cyc, double a, double b, int n) {
    double x = a + threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) x = x + b;
            else if (OP == 1) x = x * b;
            else if (OP == 2) x = fma(x, b, a);
            else if (OP == 3) x = b / x;
            else if (OP == 4) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + a; }
            else if (OP == 5) x = __shfl_xor_sync(0xffffffffu, x, 1) + b;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void smem_chain(double *out, long long *cyc, int n) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) & 1023);
    __syncthreads();
    int idx = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) idx = (int)s[idx];
    }
    long long t1 = clock64();
    out[threadIdx.x] = idx;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void bar_chain(long long *cyc, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double *out; long long *cyc;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    const int n = 256;
    const char *names[] = {"DADD", "DMUL", "DFMA", "div (IEEE /)", "MUFU.RCP64H+DADD", "SHFL+DADD"};
    for (int op = 0; op < 6; ++op) {
        long long c = 0;
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
            case 0: chain<0><<<1, 32>>>(out, cyc, 1.0, 1e-9, n); break;
            case 1: chain<1><<<1, 32>>>(out, cyc, 1.0, 1.0000001, n); break;
            case 2: chain<2><<<1, 32>>>(out, cyc, 1.0, 0.5, n); break;
            case 3: chain<3><<<1, 32>>>(out, cyc, 1.0, 1.5, n); break;
            case 4: chain<4><<<1, 32>>>(out, cyc, 1.0, 1.5, n); break;
            case 5: chain<5><<<1, 32>>>(out, cyc, 1.0, 1e-9, n); break;
            }
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-20s %.2f cycles per dependent op\n", names[op], (double)c / (n * 16));
    }
    long long c = 0;
    for (int rep = 0; rep < 2; ++rep) { smem_chain<<<1, 32>>>(out, cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); }
    printf("%-20s %.2f cycles per dependent op\n", "LDS+F2I", (double)c / (n * 16));
    for (int nt : {128, 256, 512, 1024}) {
        for (int rep = 0; rep < 2; ++rep) { bar_chain<<<1, nt>>>(cyc, 4096); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); }
        printf("__syncthreads %4d thr %.2f cycles\n", nt, (double)c / 4096);
    }
    return 0;
}
