// Per-level loop cost pieces (diagnostics): one warp, N iterations of a
// dependent level body, with or without an mbarrier try_wait / shuffles /
// shared-memory round trips / global stores, timed with clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ uint64_t bar;
    __shared__ double sm[256];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar)));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&bar)));  // phase 0 complete
    }
    sm[threadIdx.x] = 1.0;
    __syncthreads();
    double last = threadIdx.x, v0 = 0.5, v1 = 0.25, v2 = 0.125, b = 1.0;
    double* g = out + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (MODE & 1) {  // try_wait on a completed phase
            uint32_t ok;
            do {
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                             : "=r"(ok) : "r"(su(&bar)), "r"(0) : "memory");
            } while (!ok);
        }
        double left = last, down = last;
        if (MODE & 2) {
            left = __shfl_up_sync(0xffffffffu, last, 1);
            down = __shfl_up_sync(0xffffffffu, last, 8);
        }
        if (MODE & 4) {  // shared-memory edge read
            volatile double* vs = sm;
            left += vs[(threadIdx.x + i) & 255];
        }
        double acc = __dsub_rn(b, __dmul_rn(v0, last));
        acc = __dsub_rn(acc, __dmul_rn(v1, down));
        acc = __dsub_rn(acc, __dmul_rn(v2, left));
        last = acc;
        if (MODE & 8) {  // shared-memory edge write
            volatile double* vs = sm;
            vs[(threadIdx.x * 3 + i) & 255] = last;
        }
        if (MODE & 16) {  // coalesced global store
            g[(size_t)i * 32] = last;
        }
        if (MODE & 32) __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
    out[threadIdx.x] = last;
}

template <int M>
void run(double* out, long long* cyc, int n) {
    k<M><<<1, 32>>>(out, cyc, n);
    cudaDeviceSynchronize();
    printf("mode %2d (%s%s%s%s%s%s): %.1f cycles / level\n", M, (M & 1) ? "trywait " : "", (M & 2) ? "shfl " : "",
           (M & 4) ? "lds " : "", (M & 8) ? "sts " : "", (M & 16) ? "stg " : "", (M & 32) ? "syncwarp" : "",
           cyc[M] / (double)n);
}

int main() {
    double* out; long long* cyc;
    const int n = 4096;
    cudaMalloc(&out, (size_t)n * 32 * 8 + 4096);
    cudaMallocManaged(&cyc, 64 * 8);
    run<0>(out, cyc, n);
    run<1>(out, cyc, n);
    run<2>(out, cyc, n);
    run<3>(out, cyc, n);
    run<4>(out, cyc, n);
    run<8>(out, cyc, n);
    run<16>(out, cyc, n);
    run<32>(out, cyc, n);
    run<63>(out, cyc, n);
    return 0;
}
