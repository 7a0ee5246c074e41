// Latency microbenchmarks that calibrate the pipelined trisolve design on
// B200 (diagnostics only; built by `make -C tools`, run under gpurun).
//   1. cross-SM ping-pong handoff: st.release.gpu / ld.acquire.gpu, and
//      st.relaxed / ld.relaxed (volatile) variants, flags on separate lines
//   2. dependent L2-hit pointer chase (ld.global, ld.global.cg)
//   3. FP64 dependent chains: DADD, DMUL, DDIV (__ddiv_rn)
//   4. mbarrier arrive -> try_wait wake inside a CTA
//   5. bar.sync cost, 128/256 threads
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) { uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) { uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rlx(uint32_t* p, uint32_t v) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// flags[0] and flags[32] are on different 128-byte lines
template <int MODE>
__global__ void pingpong(uint32_t* flags, int iters, uint64_t* out) {
    if (threadIdx.x != 0) return;
    uint32_t* mine = flags + (blockIdx.x == 0 ? 0 : 32);
    uint32_t* other = flags + (blockIdx.x == 0 ? 32 : 0);
    const uint64_t t0 = gt();
    for (int i = 1; i <= iters; ++i) {
        if (blockIdx.x == 0) {
            if (MODE == 0) st_rel(mine, i); else st_rlx(mine, i);
            if (MODE == 0) { while (ld_acq(other) < (uint32_t)i) {} } else { while (ld_rlx(other) < (uint32_t)i) {} }
        } else {
            if (MODE == 0) { while (ld_acq(other) < (uint32_t)i) {} } else { while (ld_rlx(other) < (uint32_t)i) {} }
            if (MODE == 0) st_rel(mine, i); else st_rlx(mine, i);
        }
    }
    if (blockIdx.x == 0) out[0] = gt() - t0;
}

// handoff with a data payload written by 128 threads before the release
__global__ void pingpong_payload(uint32_t* flags, double* data, int iters, uint64_t* out) {
    uint32_t* mine = flags + (blockIdx.x == 0 ? 0 : 32);
    uint32_t* other = flags + (blockIdx.x == 0 ? 32 : 0);
    double* dmine = data + (blockIdx.x == 0 ? 0 : 4096);
    const double* dother = data + (blockIdx.x == 0 ? 4096 : 0);
    __shared__ double sink;
    const uint64_t t0 = gt();
    for (int i = 1; i <= iters; ++i) {
        if (blockIdx.x == 1 || i > 1) {
            if (threadIdx.x == 0) while (ld_acq(other) < (uint32_t)(blockIdx.x == 0 ? i - 1 : i)) {}
            __syncthreads();
            double v = dother[threadIdx.x * 8];
            if (v == -1.0) sink = v;
        }
        dmine[threadIdx.x * 8] = i;
        __syncthreads();
        if (threadIdx.x == 0) st_rel(mine, i);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gt() - t0;
}

__global__ void chase(const int* next, int steps, int start, uint64_t* out, int cg) {
    int p = start;
    const long long t0 = clock64();
    if (cg) {
        for (int i = 0; i < steps; ++i) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(p) : "l"(next + p));
    } else {
        for (int i = 0; i < steps; ++i) p = next[p];
    }
    out[0] = clock64() - t0;
    out[1] = p;
}

__global__ void fpchain(double a, double b, int n, uint64_t* out, double* sink) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(x, b);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = __dsub_rn(x, __dmul_rn(b, x));
    long long t4 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3;
    sink[0] = x;
}

__global__ void mbar_wake(int iters, uint64_t* out) {
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[1])));
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        // warp 0 arrives on bar[0], warp 1 waits it then arrives bar[1], warp 0 waits bar[1]
        uint32_t par = i & 1;
        if (w == 0) {
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[0])) : "memory");
            uint32_t ok = 0;
            while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar[1])), "r"(par) : "memory");
        } else if (w == 1) {
            uint32_t ok = 0;
            while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar[0])), "r"(par) : "memory");
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[1])) : "memory");
        }
    }
    if (threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void barsync(int iters, uint64_t* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void ldgsts_lat(const double* src, int iters, uint64_t* out) {
    __shared__ double buf[64];
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"((uint32_t)__cvta_generic_to_shared(&buf[threadIdx.x])), "l"(src + (i * 37 % 4096)) : "memory");
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    if (threadIdx.x == 0) out[0] = clock64() - t0;
}

int main() {
    uint32_t* flags; double* data; uint64_t* out; int* next; double* sink;
    CK(cudaMalloc(&flags, 4096)); CK(cudaMalloc(&data, 1 << 20)); CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&sink, 64));
    const int iters = 20000;
    uint64_t h[4];
    for (int mode = 0; mode < 2; ++mode) {
        CK(cudaMemset(flags, 0, 4096));
        if (mode == 0) pingpong<0><<<2, 32>>>(flags, iters, out); else pingpong<1><<<2, 32>>>(flags, iters, out);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        printf("pingpong %s: one-way handoff %.1f ns\n", mode == 0 ? "release/acquire.gpu" : "relaxed.gpu", h[0] / (2.0 * iters));
    }
    CK(cudaMemset(flags, 0, 4096));
    pingpong_payload<<<2, 128>>>(flags, data, iters, out);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
    printf("pingpong with 128-thread payload + bar + release: one-way %.1f ns\n", h[0] / (2.0 * iters));
    // pointer chase in a 8 MB region (L2 resident after first pass)
    const int N = 1 << 21;
    std::vector<int> hn(N);
    for (int i = 0; i < N; ++i) hn[i] = (int)((i + 40961LL * 97) % N);
    CK(cudaMalloc(&next, N * 4)); CK(cudaMemcpy(next, hn.data(), N * 4, cudaMemcpyHostToDevice));
    for (int cg = 0; cg < 2; ++cg) {
        chase<<<1, 1>>>(next, 2000, 0, out, cg); CK(cudaDeviceSynchronize());
        chase<<<1, 1>>>(next, 2000, 0, out, cg); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost));
        printf("L2-hit pointer chase (%s): %.1f cycles/load\n", cg ? "ld.cg" : "ld", h[0] / 2000.0);
    }
    fpchain<<<1, 1>>>(1.0, 1.0000001, 1000, out, sink); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
    printf("FP64 latency (cycles): dadd %.1f dmul %.1f ddiv %.1f sub(mul) %.1f\n", h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0);
    mbar_wake<<<1, 64>>>(10000, out); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
    printf("mbarrier arrive->wake round trip between warps: %.1f cycles (one way ~half)\n", h[0] / 10000.0);
    for (int t : {128, 256, 352}) {
        barsync<<<1, t>>>(10000, out); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        printf("__syncthreads %d threads: %.1f cycles\n", t, h[0] / 10000.0);
    }
    ldgsts_lat<<<1, 32>>>(data, 2000, out); CK(cudaDeviceSynchronize());
    ldgsts_lat<<<1, 32>>>(data, 2000, out); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
    printf("cp.async 8B + wait_all (L2 hit): %.1f cycles\n", h[0] / 2000.0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SM clock attr %.0f MHz\n", clk / 1000.0);
    return 0;
}
