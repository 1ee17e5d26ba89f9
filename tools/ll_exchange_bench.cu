// Latency of an all-to-all exchange of one double per CTA among G co-resident
// CTAs through global memory with LL-style flagged words (payload and epoch in
// one 8-byte store, no fence), against a release/acquire counter barrier.
//   nvcc -arch=sm_100a -O3 -o tools/exp/ll_exchange_bench tools/ll_exchange_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// mode 0: LL words; slot[parity][cta][2], each word = (epoch << 32) | half of the payload
__global__ void ll_kernel(unsigned long long *slots, int iters, int group, double *out,
                          long long *cycles, int *fail) {
    extern __shared__ double pad[];
    const int q = blockIdx.x % group, g = blockIdx.x / group;
    unsigned long long *base = slots + (size_t)g * 2 * group * 2;
    double acc = q;
    const int lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        const int par = it & 1;
        unsigned long long *s = base + par * group * 2;
        if (threadIdx.x < 32) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
            if (lane < 2)
                st_relaxed(s + q * 2 + lane, ((unsigned long long)it << 32) |
                                                 (lane ? (bits >> 32) : (bits & 0xffffffffull)));
            // lanes 0..2*group-1 poll one word each
            unsigned long long w = 0;
            if (lane < 2 * group) {
                int spins = 0;
                do {
                    w = ld_relaxed(s + lane);
                    if (++spins > 2000000) { *fail = 1; break; }
                } while ((w >> 32) != (unsigned)it);
            }
            // reassemble: max over CTAs of the payloads
            const unsigned lo = __shfl_sync(0xffffffffu, (unsigned)w, (lane & 15) * 2);
            const unsigned hi = __shfl_sync(0xffffffffu, (unsigned)w, (lane & 15) * 2 + 1);
            double v = __longlong_as_double(((long long)hi << 32) | lo);
            if ((lane & 15) >= group) v = 0.0;
            for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) pad[0] = v;
        }
        __syncthreads();
        acc = pad[0] * 0.5 + q + it;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = acc; cycles[blockIdx.x] = t1 - t0; }
}

// mode 1: data store, __threadfence, atomic counter, spin (release/acquire barrier)
__global__ void bar_kernel(double *data, unsigned long long *ctr, int iters, int group, double *out,
                           long long *cycles, int *fail) {
    extern __shared__ double pad[];
    const int q = blockIdx.x % group, g = blockIdx.x / group;
    double acc = q;
    long long t0 = clock64();
    for (int it = 1; it <= iters; ++it) {
        const int par = it & 1;
        double *d = data + ((size_t)g * 2 + par) * group;
        if (threadIdx.x == 0) {
            d[q] = acc;
            __threadfence();
            atomicAdd(ctr + g, 1ull);
            int spins = 0;
            while (*((volatile unsigned long long *)(ctr + g)) < (unsigned long long)it * group)
                if (++spins > 2000000) { *fail = 1; break; }
            __threadfence();
            double v = 0.0;
            for (int j = 0; j < group; ++j) v = fmax(v, ((volatile double *)d)[j]);
            pad[0] = v;
        }
        __syncthreads();
        acc = pad[0] * 0.5 + q + it;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = acc; cycles[blockIdx.x] = t1 - t0; }
}

int main() {
    const int iters = 2000;
    for (int group : {2, 4, 8, 16}) {
        for (int ngroups : {1, 9}) {
            if (group * ngroups > 148) continue;
            const int n = group * ngroups;
            unsigned long long *slots, *ctr;
            double *out, *data;
            long long *cyc;
            int *fail;
            cudaMalloc(&slots, sizeof(unsigned long long) * ngroups * 2 * group * 2);
            cudaMemset(slots, 0, sizeof(unsigned long long) * ngroups * 2 * group * 2);
            cudaMalloc(&ctr, 8 * ngroups);
            cudaMalloc(&data, 8 * ngroups * 2 * group);
            cudaMalloc(&out, 8 * n);
            cudaMalloc(&cyc, 8 * n);
            cudaMalloc(&fail, 4);
            cudaMemset(fail, 0, 4);
            cudaFuncSetAttribute(ll_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
            cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
            for (int mode = 0; mode < 2; ++mode) {
                cudaMemset(ctr, 0, 8 * ngroups);
                cudaMemset(slots, 0, sizeof(unsigned long long) * ngroups * 2 * group * 2);
                void *args0[] = {&slots, (void *)&iters, &group, &out, &cyc, &fail};
                void *args1[] = {&data, &ctr, (void *)&iters, &group, &out, &cyc, &fail};
                cudaError_t e = cudaLaunchCooperativeKernel(
                    mode == 0 ? (void *)ll_kernel : (void *)bar_kernel, dim3(n), dim3(128),
                    mode == 0 ? args0 : args1, 150 * 1024, 0);
                cudaError_t e2 = cudaDeviceSynchronize();
                long long h[148];
                int hf = 0;
                cudaMemcpy(h, cyc, 8 * n, cudaMemcpyDeviceToHost);
                cudaMemcpy(&hf, fail, 4, cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < n; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("group %2d x %d groups  %s  %.0f cycles/exchange  (launch %d sync %d fail %d)\n",
                       group, ngroups, mode == 0 ? "LL words      " : "fence+counter ",
                       (double)mx / iters, (int)e, (int)e2, hf);
            }
            cudaFree(slots); cudaFree(ctr); cudaFree(data); cudaFree(out); cudaFree(cyc); cudaFree(fail);
        }
    }
    return 0;
}
