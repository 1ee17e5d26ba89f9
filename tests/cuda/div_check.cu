// Test helper (not product code): checks mgp::div_shared against the
// compiler's IEEE a / b on random and edge-case operands.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_2104_09404_b200/csrc/div_shared.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}

__device__ double pick(uint64_t h, int mode) {
    if (mode == 0) {  // any bit pattern (includes NaN/inf/denormals/zeros)
        return __longlong_as_double((long long)h);
    }
    if (mode == 1) {  // realistic WENO ranges: raw in [1e-30, 1e15], S >= raw
        const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
        return exp2(-100.0 + 150.0 * u);
    }
    // exponent extremes
    const uint64_t ex = (h >> 52) & 0x7ff;
    const uint64_t e2 = (ex & 1) ? (ex & 0x3f) : (0x7ff - (ex & 0x3f));
    return __longlong_as_double((long long)((h & 0x800fffffffffffffull) | (e2 << 52)));
}

__global__ void div_kernel(uint64_t seed, int64_t n, int mode, unsigned long long *bad,
                           double *witness) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t h1 = mix(seed ^ (2 * i + 1)), h2 = mix(seed * 31 + 2 * i);
    const double b = pick(h2, mode);
    const mgp::SharedRcp R = mgp::shared_rcp(b);
    for (int j = 0; j < 3; ++j) {
        const double a = pick(mix(h1 + j), mode);
        const double want = a / b;
        const double got = mgp::div_shared(a, R);
        bool flag = false;
        const double fast = mgp::div_fast(a, R, flag);
        const bool same = __double_as_longlong(want) == __double_as_longlong(got) ||
                          (want != want && got != got);
        const bool fast_ok = flag || __double_as_longlong(want) == __double_as_longlong(fast) ||
                             (want != want && fast != fast);
        if (!same || !fast_ok) {
            if (atomicAdd(bad, 1ull) == 0) {
                witness[0] = a; witness[1] = b; witness[2] = want; witness[3] = got;
            }
        }
    }
}

extern "C" int64_t div_check(uint64_t seed, int64_t n, int mode, double *witness_host) {
    unsigned long long *bad;
    double *w;
    cudaMalloc(&bad, sizeof(*bad));
    cudaMalloc(&w, 4 * sizeof(double));
    cudaMemset(bad, 0, sizeof(*bad));
    cudaMemset(w, 0, 4 * sizeof(double));
    div_kernel<<<(unsigned)((n + 255) / 256), 256>>>(seed, n, mode, bad, w);
    unsigned long long h = 0;
    cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(witness_host, w, 4 * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(bad);
    cudaFree(w);
    return cudaGetLastError() == cudaSuccess ? (int64_t)h : -1;
}
