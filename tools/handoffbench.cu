// Intra-CTA warp-to-warp handoff: data in shared memory + progress signal
// (diagnostics for the wave kernel's cross-warp dependencies).
//   A: STS data; __syncwarp; fence.acq_rel.cta; STS flag  <->  volatile LDS spin
//   B: STS data; mbarrier.arrive (all 32 lanes)          <->  try_wait.parity
//   C: STS data; __syncwarp; STS flag (no fence)          <->  volatile LDS spin
// Warp 0 and warp 1 ping-pong; NBUSY other warps keep issuing STS/LDS traffic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MODE>
__global__ void hb(int iters, int busy_warps, long long* out, double* sink) {
    __shared__ double data[2][32];
    __shared__ volatile uint32_t flag[2];
    __shared__ __align__(8) uint64_t bar[2][64];
    __shared__ double scratch[16][64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        flag[0] = flag[1] = 0;
        for (int i = 0; i < 64; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[0][i])), "r"(32));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[1][i])), "r"(32));
        }
    }
    __syncthreads();
    if (warp >= 2) {  // background load
        if (warp - 2 >= busy_warps) return;
        double acc = 0;
        for (int i = 0; i < iters * 8; ++i) {
            scratch[warp & 15][(i + lane) & 63] = acc;
            acc += scratch[warp & 15][(i * 7 + lane) & 63];
        }
        sink[threadIdx.x] = acc;
        return;
    }
    const int me = warp, other = warp ^ 1;
    long long t0 = clock64();
    double v = lane;
    for (int i = 0; i < iters; ++i) {
        // wait for the other warp's round i (warp 0 starts)
        if (!(me == 0 && i == 0)) {
            const int k = me == 0 ? i - 1 : i;  // round the other warp published
            if (MODE == 1) {
                uint32_t ok = 0;
                const uint32_t par = (k >> 6) & 1;
                while (!ok)
                    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                                 : "=r"(ok) : "r"(sa(&bar[other][k & 63])), "r"(par) : "memory");
            } else {
                while (flag[other] < (uint32_t)(k + 1)) {}
            }
            v += data[other][lane];
        }
        data[me][lane] = v;
        if (MODE == 1) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[me][i & 63])) : "memory");
        } else {
            __syncwarp();
            if (MODE == 0) asm volatile("fence.acq_rel.cta;" ::: "memory");
            if (lane == 0) flag[me] = i + 1;
        }
    }
    if (threadIdx.x == 0) out[0] = (clock64() - t0) / (2 * iters);
    sink[threadIdx.x] = v;
}
int main() {
    long long* out; double* sink; long long h;
    cudaMalloc(&out, 8); cudaMalloc(&sink, 8192);
    const char* nm[] = {"fence + flag", "mbarrier arrive/try_wait", "flag, no fence"};
    for (int busy : {0, 14}) for (int m = 0; m < 3; ++m) {
        for (int r = 0; r < 2; ++r) {
            if (m == 0) hb<0><<<1, 512>>>(60, busy, out, sink);
            if (m == 1) hb<1><<<1, 512>>>(60, busy, out, sink);
            if (m == 2) hb<2><<<1, 512>>>(60, busy, out, sink);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("busy warps %2d  %-26s one-way %lld cycles\n", busy, nm[m], h);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
