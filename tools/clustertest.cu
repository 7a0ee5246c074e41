// Can the wave kernel's launch shape run as clusters (diagnostics)? Queries the
// max active clusters for cluster sizes 2/4/8 at ~220 KB dynamic shared memory
// per CTA, then does a cooperative cluster launch of 148 CTAs with a DSMEM
// ping between cluster peers and reports the round trip.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void kern(long long* out, int iters) {
    extern __shared__ __align__(16) unsigned char sm[];
    volatile unsigned* flag = reinterpret_cast<volatile unsigned*>(sm);
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) flag[0] = 0;
    cl.sync();
    const unsigned rank = cl.block_rank();
    unsigned* peer = cl.map_shared_rank(reinterpret_cast<unsigned*>(sm), rank ^ 1);
    if (threadIdx.x == 0 && blockIdx.x < 2) {
        long long t0 = clock64();
        for (int i = 1; i <= iters; ++i) {
            if (rank == 0) {
                asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"l"(peer), "r"((unsigned)i) : "memory");
                while (flag[0] != 2u * i) {}
            } else {
                while (flag[0] != (unsigned)i) {}
                asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"l"(peer), "r"(2u * i) : "memory");
            }
        }
        if (rank == 0) out[0] = (clock64() - t0) / iters;
    }
    cl.sync();
}
int main() {
    const int smem = 220 * 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(640); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int nc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs) %s\n", cs, nc, nc * cs, cudaGetErrorString(e));
    }
    long long* out; long long h = 0; cudaMalloc(&out, 8);
    for (int cs : {2}) {
        for (int grid : {148, 146, 144}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid); cfg.blockDim = dim3(640); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
            cfg.attrs = at; cfg.numAttrs = 2;
            int iters = 1000;
            cudaError_t e = cudaLaunchKernelEx(&cfg, kern, out, iters);
            cudaError_t e2 = cudaDeviceSynchronize();
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("cooperative cluster launch cs=%d grid=%d: %s / %s, DSMEM round trip %lld cycles\n", cs, grid, cudaGetErrorString(e), cudaGetErrorString(e2), h);
        }
    }
}
