// One-way cross-SM handoff latency of mailbox store/load flavours (diagnostics).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
template <int MODE> __device__ __forceinline__ void put(u64* p, u64 v) {
    if (MODE == 0) asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v), "l"(v) : "memory");
    if (MODE == 1) { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
                     asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p + 1), "l"(v) : "memory"); }
    if (MODE == 2) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 3) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 4) asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 5) asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v), "l"(v) : "memory");
}
template <int MODE> __device__ __forceinline__ bool got(const u64* p, u64 v) {
    u64 a, b = v;
    if (MODE == 0) asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if (MODE == 1) { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
                     asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(b) : "l"(p + 1) : "memory"); }
    if (MODE == 2) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
    if (MODE == 3) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
    if (MODE == 4) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
    if (MODE == 5) asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    return a == v && b == v;
}
template <int MODE> __global__ void pp(u64* box, int iters, long long* out) {
    if (threadIdx.x) return;
    u64* mine = box + (blockIdx.x ? 0 : 32);
    u64* other = box + (blockIdx.x ? 32 : 0);
    long long t0 = clock64();
    for (u64 i = 1; i <= (u64)iters; ++i) {
        if (blockIdx.x == 0) { put<MODE>(other, i); while (!got<MODE>(mine, i)) {} }
        else { while (!got<MODE>(mine, i)) {} put<MODE>(other, i); }
    }
    if (blockIdx.x == 0) out[MODE] = (clock64() - t0) / (2 * iters);
}
int main() {
    long long* out; u64* box; long long h[8];
    cudaMalloc(&out, 64); cudaMalloc(&box, 4096);
    const char* nm[] = {"relaxed v2.u64", "relaxed 2x u64", "relaxed u64", "volatile u64", "cg u64", "cg v2.u64"};
    for (int r = 0; r < 2; ++r) {
#define RUN(M) cudaMemset(box, 0, 4096); pp<M><<<2, 32>>>(box, 2000, out); cudaDeviceSynchronize();
        RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
    }
    cudaMemcpy(h, out, 48, cudaMemcpyDeviceToHost);
    for (int m = 0; m < 6; ++m) printf("%-16s one-way %lld cycles\n", nm[m], h[m]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
