// Latency microbenchmarks (diagnostics): dependent chains timed with clock64 on one warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double seed, int n) {
    __shared__ double sm[64];
    __shared__ unsigned long long bar;
    double a = seed + threadIdx.x, b = 1.0000001;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = __fma_rn(a, b, 1e-300);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // SHFL (double) chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) a = __shfl_up_sync(0xffffffffu, a, 1) + 0.0;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // LDS/STS chain through shared memory
    sm[threadIdx.x % 64] = a;
    __syncwarp();
    volatile double* vs = sm;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double v = vs[(threadIdx.x + i) % 64]; vs[(threadIdx.x + i + 1) % 64] = v + 0.0; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // named barrier among all warps of the block
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = t1 - t0;
    out[threadIdx.x] = a;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMallocManaged(&cyc, 64 * 8);
    const int n = 1000;
    for (int threads : {32, 128, 512}) {
        k<<<1, threads>>>(out, cyc, 1.0, n);
        cudaDeviceSynchronize();
        printf("threads %3d: per op cycles: DADD %.1f DMUL %.1f DFMA %.1f SHFL.f64(+DADD) %.1f LDS+STS(+DADD) %.1f bar.sync %.1f\n",
               threads, cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n, cyc[3] / (double)n,
               cyc[4] / (double)n, cyc[5] / (double)n);
    }
    return 0;
}
