// Per-chunk cost of the wave solver's group handoff in isolation (diagnostics).
// K warps take "chunks" round robin; chunk j waits (named barrier 1 + j % K,
// 64 threads) for chunk j-1, reads its value from shared memory, does the row
// arithmetic and releases chunk j+1. Variants add the kernel's other per-chunk
// work one piece at a time. Prints cycles per chunk.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void bsync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void barv(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(sa(b)) : "memory"); }
__device__ __noinline__ double div_slow(double a, double d) { return __ddiv_rn(a, d); }

template <int K, int V>
__global__ void __launch_bounds__(32 * K) chain(int nch, double* xs, unsigned long long* mbox, long long* out) {
    __shared__ double ring[2048];
    __shared__ double rowdata[2048];
    __shared__ uint64_t bars[16];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) { ring[i] = 1.0; rowdata[i] = 4.0 + (i & 7); }
    if (threadIdx.x == 0) for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    __syncthreads();
    long long t0 = clock64();
    for (int j = w; j < nch; j += K) {
        // prep (independent of the chain)
        const double dv = rowdata[(j * 32 + lane) & 2047];
        const double y = __drcp_rn(dv);
        const double v = 0.25, b = 1.0;
        const int src = ((j - 1) * 32 + lane) & 2047;
        if (j > 0) bsync(1 + j % K, 64);
        const double xv = ring[src];
        const double a = __dsub_rn(b, __dmul_rn(v, xv));
        double x;
        if (V & 1) {
            const double q = __dmul_rn(a, y); const double r = __fma_rn(-dv, q, a); x = __fma_rn(r, y, q);
            const double aa = fabs(a), aq = fabs(x);
            if (!(aa > 0x1p-900 && aa < 0x1p900 && aq > 0x1p-900 && aq < 0x1p900)) x = div_slow(a, dv);
        } else {
            x = a * 0.25;
        }
        if (V & 2) {  // mailbox store (relaxed gpu, 16 B) by every lane
            unsigned long long bits = (unsigned long long)__double_as_longlong(x);
            asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(mbox + 2 * ((j * 32 + lane) & 1048575)), "l"(bits), "l"(bits) : "memory");
        }
        ring[(j * 32 + lane) & 2047] = x;
        if (j + 1 < nch) barv(1 + (j + 1) % K, 64);
        if ((V & 4) && lane == 0) mbar_arrive(&bars[j & 15]);
        if (V & 8) xs[(size_t)((j * 32 + lane) * 977) & ((1 << 24) - 1)] = x;  // scattered x store
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
    double* xs; unsigned long long* mbox; long long* out; long long h;
    cudaMalloc(&xs, 8 << 24); cudaMalloc(&mbox, 16 << 20); cudaMalloc(&out, 8);
    const int nch = 20000;
    auto run = [&](auto kern, const char* name, int K) {
        for (int r = 0; r < 2; ++r) kern<<<1, 32 * K>>>(nch, xs, mbox, out);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("K=%d %-40s %7.1f cycles/chunk\n", K, name, (double)h / nch);
    };
    run(chain<4, 0>, "barrier + LDS + mul", 4);
    run(chain<4, 1>, "+ Markstein", 4);
    run(chain<4, 3>, "+ mailbox st.relaxed.gpu", 4);
    run(chain<4, 7>, "+ mbarrier arrive", 4);
    run(chain<4, 15>, "+ scattered x STG", 4);
    run(chain<8, 0>, "barrier + LDS + mul", 8);
    run(chain<8, 15>, "all", 8);
    run(chain<2, 0>, "barrier + LDS + mul", 2);
    run(chain<2, 15>, "all", 2);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
