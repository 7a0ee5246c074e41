// Producer-loop cost of the wave kernel in isolation (diagnostics): one warp
// issues cp.async.bulk copies of chunk-sized pieces into a shared-memory ring
// (mbarrier complete_tx), one consumer warp waits each chunk and releases its
// slot. Prints cycles per chunk for several copy shapes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) { while (!try_wait(b, par)) {} }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) { asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(sa(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
template <int MODE>
__global__ void tb(const char* g, int nch, int bytes, long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 16;
    unsigned char* buf = sm + 1024;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int s = 0; s < 16; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    long long t0 = clock64();
    if (warp == 0) {
        for (int j = 0; j < nch; ++j) {
            const int s = j & 15;
            if (lane == 0) {
                if (j >= 16) wait(&empty[s], ((j >> 4) - 1) & 1);
                unsigned char* dst = buf + s * 8192;
                const char* src = g + (size_t)j * 8192 % (1 << 26);
                if (MODE == 0) { expect_tx(&full[s], 0); }
                if (MODE == 1) { expect_tx(&full[s], bytes); bulk(dst, src, bytes, &full[s]); }
                if (MODE == 2) { expect_tx(&full[s], bytes + 256); bulk(dst + 512, src, bytes, &full[s]); bulk(dst, src + (1 << 25), 256, &full[s]); }
            }
            __syncwarp();
        }
    } else {
        for (int j = 0; j < nch; ++j) {
            const int s = j & 15;
            wait(&full[s], (j >> 4) & 1);
            __syncwarp();
            if (lane == 0) arrive(&empty[s]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
}
int main() {
    char* g; long long* out; long long h;
    cudaMalloc(&g, 1 << 27); cudaMalloc(&out, 8);
    const int nch = 20000, smem = 1024 + 16 * 8192;
    auto run = [&](auto k, const char* nm, int bytes) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int r = 0; r < 2; ++r) k<<<1, 64, smem>>>(g, nch, bytes, out);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("%-34s bytes %5d  %7.1f cycles/chunk\n", nm, bytes, (double)h / nch);
    };
    run(tb<0>, "arrive.expect_tx only", 0);
    for (int b : {1024, 4096, 8192 - 512}) run(tb<1>, "1 bulk copy", b);
    for (int b : {1024, 4096}) run(tb<2>, "2 bulk copies", b);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
