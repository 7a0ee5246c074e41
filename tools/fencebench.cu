// Cost of CTA-scope ordering primitives with global traffic in flight
// (diagnostics for the wave trisolve's per-chunk publish step).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void fb(double* g, const double* src, int iters, long long* out) {
    __shared__ double sh[1024];
    __shared__ volatile uint32_t flag[32];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        sh[(i * 32 + lane) & 1023] = i;
        if (MODE == 1 || MODE == 2 || MODE == 5) g[(size_t)i * 4096 + lane * 37] = i;       // global store in flight
        if (MODE == 3 || MODE == 4) {                                     // cp.async gather in flight
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(&sh[(i * 32 + lane + 512) & 1023])),
                         "l"(src + ((size_t)i * 4099 + lane * 1031) % (1 << 24)) : "memory");
        }
        __syncwarp();
        if (MODE == 0 || MODE == 1 || MODE == 3) __threadfence_block();
        if (MODE == 5) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) flag[0] = i;
    }
    if (threadIdx.x == 0) out[MODE] = clock64() - t0;
}

int main() {
    double *g, *src; long long* out; long long h[8];
    cudaMalloc(&g, (size_t)8 << 27); cudaMalloc(&src, (size_t)8 << 24); cudaMalloc(&out, 64);
    const int iters = 2000;
    const char* names[] = {"STS + fence.cta", "STS + STG + fence.cta", "STS + STG, no fence", "STS + cp.async + fence.cta",
                           "STS + cp.async, no fence", "STS + STG + fence.proxy.async"};
    for (int rep = 0; rep < 2; ++rep) {
        fb<0><<<1, 32>>>(g, src, iters, out); fb<1><<<1, 32>>>(g, src, iters, out); fb<2><<<1, 32>>>(g, src, iters, out);
        fb<3><<<1, 32>>>(g, src, iters, out); fb<4><<<1, 32>>>(g, src, iters, out); fb<5><<<1, 32>>>(g, src, iters, out);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(h, out, 48, cudaMemcpyDeviceToHost);
    for (int m = 0; m < 6; ++m) printf("%-36s %.1f cycles/iter\n", names[m], (double)h[m] / iters);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
