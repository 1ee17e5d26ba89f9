// Probe: device -> mapped pinned host write bandwidth (zero-copy) by store
// width, and the copy engine's D2H / H2D for comparison.  16.8 MB, the C2
// trajectory of one relaxation.
#include <cstdio>
#include <cuda_runtime.h>

template <int W>
__global__ void wr(double *dst, const double *src, size_t n) {
    const size_t i0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
    const size_t stride = (size_t)gridDim.x * blockDim.x * W;
    for (size_t i = i0; i < n; i += stride) {
        if (W == 1) dst[i] = src[i];
        if (W == 2) reinterpret_cast<double2 *>(dst)[i / 2] = reinterpret_cast<const double2 *>(src)[i / 2];
        if (W == 4) {
            const double4 v = reinterpret_cast<const double4 *>(src)[i / 4];
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + i), "d"(v.x), "d"(v.y),
                         "d"(v.z), "d"(v.w) : "memory");
        }
    }
}

int main() {
    const size_t n = 4097 * 512;   // rows x cells
    double *h, *hd, *d;
    cudaHostAlloc(&h, n * 8, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaMalloc(&d, n * 8);
    cudaMemset(d, 0, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    const int grids[] = {148, 592, 1184};
    const int thr[] = {128, 256};
    for (int g : grids)
        for (int t : thr) {
            for (int w = 1; w <= 4; w *= 2) {
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    for (int k = 0; k < 10; ++k) {
                        if (w == 1) wr<1><<<g, t>>>(hd, d, n);
                        if (w == 2) wr<2><<<g, t>>>(hd, d, n);
                        if (w == 4) wr<4><<<g, t>>>(hd, d, n);
                    }
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    cudaEventElapsedTime(&ms, a, b);
                }
                printf("zero-copy write grid %4d x %3d, %2d B stores: %6.1f GB/s\n", g, t, 8 * w,
                       10.0 * n * 8 / (ms * 1e-3) / 1e9);
            }
        }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        for (int k = 0; k < 10; ++k) cudaMemcpyAsync(h, d, n * 8, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    printf("copy engine D2H: %6.1f GB/s\n", 10.0 * n * 8 / (ms * 1e-3) / 1e9);
    cudaEventRecord(a);
    for (int k = 0; k < 10; ++k) cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("copy engine H2D: %6.1f GB/s\n", 10.0 * n * 8 / (ms * 1e-3) / 1e9);
    return 0;
}
