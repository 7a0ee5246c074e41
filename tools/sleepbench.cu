// __nanosleep granularity and v2 relaxed mailbox one-way latency between two SMs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void sl(int ns, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < 100; ++i) __nanosleep(ns);
    out[0] = (clock64() - t0) / 100;
}
__global__ void pp(unsigned long long* box, int iters, long long* out) {
    if (threadIdx.x) return;
    unsigned long long* mine = box + (blockIdx.x ? 0 : 16);
    unsigned long long* other = box + (blockIdx.x ? 16 : 0);
    long long t0 = clock64();
    for (unsigned i = 1; i <= (unsigned)iters; ++i) {
        if (blockIdx.x == 0) {
            asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(other), "l"((unsigned long long)i << 32), "l"((unsigned long long)i << 32) : "memory");
            unsigned long long a, b;
            do { asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(mine) : "memory"); } while ((a >> 32) != i || (b >> 32) != i);
        } else {
            unsigned long long a, b;
            do { asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(mine) : "memory"); } while ((a >> 32) != i || (b >> 32) != i);
            asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(other), "l"((unsigned long long)i << 32), "l"((unsigned long long)i << 32) : "memory");
        }
    }
    if (blockIdx.x == 0) out[1] = (clock64() - t0) / (2 * iters);
}
int main() {
    long long* out; unsigned long long* box; long long h[2];
    cudaMalloc(&out, 16); cudaMalloc(&box, 4096); cudaMemset(box, 0, 4096);
    for (int ns : {0, 32, 100, 500, 1000}) {
        sl<<<1, 32>>>(ns, out); cudaDeviceSynchronize(); cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
        printf("__nanosleep(%d): %lld cycles\n", ns, h[0]);
    }
    for (int r = 0; r < 2; ++r) { cudaMemset(box, 0, 4096); pp<<<2, 32>>>(box, 2000, out); cudaDeviceSynchronize(); }
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("v2 relaxed mailbox one-way: %lld cycles\n", h[1]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
