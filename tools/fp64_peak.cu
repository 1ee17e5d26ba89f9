// fp64_peak.cu -- FP64 CUDA-core throughput probe (not part of the product
// ABI; used by bench.py to state the roofline denominator for the FP64-bound
// propagator kernels).  Independent DADD / DMUL chains (no FMA: the parity
// build runs with -fmad=false) over every SM; one op = 1 flop.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(512) fp64_addmul(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x0 = x0 * a; x1 = x1 + b; x2 = x2 * a; x3 = x3 + b;
            x4 = x4 * a; x5 = x5 + b; x6 = x6 * a; x7 = x7 + b;
        }
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(512) fp64_fma(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[blockIdx.x] = s;
}

extern "C" {
// Runs the probe; returns ops per second (1 op = one DADD/DMUL, or one DFMA
// instruction when fma != 0) measured with CUDA events, or -1 on error.
double fp64_probe(int fma, int iters) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *out = nullptr;
    if (cudaMalloc(&out, sizeof(double) * sms * 8) != cudaSuccess) return -1;
    const int blocks = sms * 4, threads = 512;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (fma) fp64_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        else fp64_addmul<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * iters * 64.0;
        const double rate = ops / (ms * 1e-3);
        if (rep > 0 && rate > best) best = rate;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? best : -1;
}
}
