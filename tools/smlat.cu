// Cross-SM ping-pong latency through L2 by SM-id pair (diagnostics): CTA on SM 0
// and CTA on SM k bounce a counter 1000 times (st/ld.relaxed.gpu). Prints the
// round-trip cycles per k, to see the die / GPC structure of SM ids.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned ldr(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void str(unsigned* p, unsigned v) { asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

__global__ void k(unsigned* flags, long long* out, int partner, int iters) {
    __shared__ int role;
    if (threadIdx.x == 0) {
        const unsigned s = smid();
        role = s == 0 ? 0 : (s == (unsigned)partner ? 1 : -1);
    }
    __syncthreads();
    if (role < 0 || threadIdx.x != 0) return;
    unsigned* ping = flags;
    unsigned* pong = flags + 32;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (role == 0) {
            str(ping, i);
            while (ldr(pong) != (unsigned)i) {}
        } else {
            while (ldr(ping) != (unsigned)i) {}
            str(pong, i);
        }
    }
    if (role == 0) out[0] = (clock64() - t0) / iters;
}
int main(int argc, char** argv) {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* flags; long long* out; long long h;
    cudaMalloc(&flags, 1 << 26); cudaMalloc(&out, 8);
    if (argc > 1) {  // fixed SM pair, flag location varied over 64 MB: does the address's home matter?
        int p = atoi(argv[1]);
        for (size_t off = 0; off < (1u << 26) - 4096; off += (1u << 26) / 32) {
            unsigned* f = flags + off / 4;
            cudaMemset(f, 0, 4096); cudaMemset(out, 0, 8);
            int iters = 1000;
            void* args[] = {&f, &out, &p, &iters};
            cudaLaunchCooperativeKernel((void*)k, dim3(sms), dim3(32), args, 0, 0);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("SM0<->SM%d flag at +%zu MB: %lld cycles\n", p, off >> 20, h);
        }
        return 0;
    }
    printf("SMs %d\n", sms);
    for (int p = 1; p < sms; ++p) {
        cudaMemset(flags, 0, 4096); cudaMemset(out, 0, 8);
        void* args[] = {&flags, &out, &p, nullptr};
        int iters = 1000; args[3] = &iters;
        cudaLaunchCooperativeKernel((void*)k, dim3(sms), dim3(32), args, 0, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("%d:%lld ", p, h);
        if (p % 12 == 0) printf("\n");
    }
    printf("\n%s\n", cudaGetErrorString(cudaGetLastError()));
}
