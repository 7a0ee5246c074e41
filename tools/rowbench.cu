// Floor of the pipelined solver's per-chunk critical path on B200, measured in
// isolation (diagnostics). One CTA; warp 1 pre-arrives every chunk barrier;
// 128 solver threads run the chunk loop on shared-memory data:
//   wait mbarrier -> header -> b -> 3 x (dep -> x) -> FP chain -> div ->
//   [stores] -> bar.sync -> arrive
// Variants switch the stores / division off to attribute the cost.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
}

template <int VARIANT>
__global__ void rowbench(int chunks, double* gx, unsigned long long* mbox, long long* out) {
    __shared__ uint64_t bar[64];
    __shared__ double ring[4096];
    __shared__ int dep[3 * 128];
    __shared__ double val[3 * 128], bst[128], diag[128];
    __shared__ int hdr[24];
    const int tid = threadIdx.x;
    if (tid == 0) for (int s = 0; s < 64; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
    for (int i = tid; i < 4096; i += blockDim.x) ring[i] = 1.0 + i * 1e-9;
    for (int i = tid; i < 384; i += blockDim.x) { dep[i] = -((i * 37) % 3000) - 1; val[i] = 0.25; }
    for (int i = tid; i < 128; i += blockDim.x) { bst[i] = 3.0; diag[i] = 4.0 + i; }
    if (tid < 24) hdr[tid] = tid == 0 ? 56 : 3;
    __syncthreads();
    if (tid >= 128 && tid < 160) {  // "waiter": arrive all chunk barriers ahead of time
        for (int j = 0; j < chunks; ++j) {
            if (j >= 64) wait(&bar[j % 64], 0), (void)0;  // never reached for chunks <= 64
            if ((tid & 31) == 0) arrive(&bar[j % 64]);
        }
        return;
    }
    if (tid >= 128) return;
    long long t0 = clock64();
    for (int j = 0; j < chunks; ++j) {
        wait(&bar[j % 64], (j / 64) & 1);
        const int m = hdr[0];
        if (tid < m) {
            double acc = bst[tid];
            double xv[3], vv[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) { xv[u] = ring[-dep[u * 128 + tid] - 1]; vv[u] = val[u * 128 + tid]; }
#pragma unroll
            for (int u = 0; u < 3; ++u) acc = __dsub_rn(acc, __dmul_rn(vv[u], xv[u]));
            double x = VARIANT == 1 ? acc : __ddiv_rn(acc, diag[tid]);
            ring[(j * 56 + tid) & 4095] = x;
            if (VARIANT >= 2) gx[j * 128 + tid] = x;
            if (VARIANT >= 3) asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(mbox + j * 128 + tid), "l"(__double_as_longlong(x)) : "memory");
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    if (tid == 0) out[0] = clock64() - t0;
}

int main() {
    double* gx; unsigned long long* mb; long long* out; long long h;
    cudaMalloc(&gx, 64 * 128 * 8); cudaMalloc(&mb, 64 * 128 * 8); cudaMalloc(&out, 8);
    const int chunks = 64;
    const char* names[] = {"div + ring store", "no div", "div + ring + STG x", "div + ring + STG x + st.relaxed mailbox"};
    for (int v = 0; v < 4; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) rowbench<0><<<1, 160>>>(chunks, gx, mb, out);
            if (v == 1) rowbench<1><<<1, 160>>>(chunks, gx, mb, out);
            if (v == 2) rowbench<2><<<1, 160>>>(chunks, gx, mb, out);
            if (v == 3) rowbench<3><<<1, 160>>>(chunks, gx, mb, out);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("%-45s %.1f cycles / chunk\n", names[v], (double)h / chunks);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
