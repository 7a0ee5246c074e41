// B200 (sm_100a) triangular-solve kernels on the HEC layouts of tri_plan.hpp.
//
// Reference semantics: hec::solve, proj/src/triangular.cpp:90-135 (Algorithm 2
// of arXiv 1606.00541). Per row: acc = b; acc -= v * x[dep] in stored order;
// x = acc / diag. Every product and difference is rounded separately
// (__dmul_rn/__dsub_rn: no FMA contraction, like the reference's mulsd/subsd)
// and the division is the IEEE-correct __ddiv_rn, so results are bitwise equal
// to the reference for any schedule.
//
// Two strategies:
//  * k_level_rows   one launch per level, thread per reordered row (baseline;
//                   the reference's level barrier becomes a kernel boundary).
//  * k_wave         persistent wavefront, one CTA per SM (wave_kernel.cuh,
//                   layout in tri_plan.hpp). Warp roles: 2 producers (bulk
//                   copies of chunk blobs into a host-placed shared-memory byte
//                   ring), 5 waiters (poll the epoch-tagged mailboxes of values
//                   from other CTAs, stage them, publish the chunk on an
//                   mbarrier), K groups of G solver warps taking the chunks round
//                   robin with a named-barrier handoff. The reference's per-level
//                   barrier becomes dataflow; no grid barrier.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "wave_kernel.cuh"

namespace hec::dev {

// -------------------------------------------------------------- LEVELS ----
// IEEE row update, never contracted into an FMA.
__device__ __forceinline__ double sub_prod(double acc, double v, double x) {
    return __dsub_rn(acc, __dmul_rn(v, x));
}

// The level kernels of one solve read their argument block from device memory,
// so the whole sequence of launches is captured once in a CUDA graph per stream
// and replayed for any vectors: one argument-setting kernel + one graph launch
// per solve instead of one launch per level.
__global__ void k_level_rows(const LevelArgs* __restrict__ pa, int r0, int r1) {
    const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    const LevelArgs& a = *pa;
    double acc = a.b[a.b_ordered ? r : a.bidx[r]];
    for (int k = 0; k < a.width; ++k) {
        const size_t slot = static_cast<size_t>(k) * a.ld + r;
        const int d = a.ell_dep[slot];
        if (d >= 0) acc = sub_prod(acc, a.ell_val[slot], a.xs[d]);
    }
    for (int t = a.tail_rp[r]; t < a.tail_rp[r + 1]; ++t) acc = sub_prod(acc, a.tail_val[t], a.xs[a.tail_dep[t]]);
    const double x = __ddiv_rn(acc, a.diag[r]);
    a.xs[a.xidx[r]] = x;
    if (a.out) {
        const int o = a.oidx[r];
        if (o >= 0) a.out[o] = x;
    }
}

__global__ void k_set_level_args(LevelArgs a, LevelArgs* dst) { *dst = a; }

void set_level_args(const LevelArgs& a, LevelArgs* dev, cudaStream_t st) {
    k_set_level_args<<<1, 1, 0, st>>>(a, dev);
}

void launch_levels(const LevelArgs* dev_args, const int* level_starts_host, int nlev, cudaStream_t st) {
    for (int k = 0; k < nlev; ++k) {
        const int r0 = level_starts_host[k], r1 = level_starts_host[k + 1];
        const int m = r1 - r0;
        const int tpb = m >= 256 ? 256 : (m >= 128 ? 128 : 64);
        k_level_rows<<<(m + tpb - 1) / tpb, tpb, 0, st>>>(dev_args, r0, r1);
    }
}


// bp[r] = b[bidx[r]]: four rows per thread (one 16-byte index load, four
// independent gathers in flight, two 16-byte stores); bidx and bp 16-byte aligned.
__global__ void __launch_bounds__(256) k_permute_in4(const double* __restrict__ b, const int* __restrict__ bidx,
                                                     double* __restrict__ bp, int n) {
    const int n4 = n >> 2;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += gridDim.x * blockDim.x) {
        const int4 i = __ldcs(reinterpret_cast<const int4*>(bidx) + q);
        const double v0 = __ldg(b + i.x), v1 = __ldg(b + i.y), v2 = __ldg(b + i.z), v3 = __ldg(b + i.w);
        __stcs(reinterpret_cast<double2*>(bp) + 2 * q, make_double2(v0, v1));
        __stcs(reinterpret_cast<double2*>(bp) + 2 * q + 1, make_double2(v2, v3));
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        const int r = 4 * n4 + threadIdx.x;
        bp[r] = __ldg(b + bidx[r]);
    }
}

__global__ void k_permute_in(const double* __restrict__ b, const int* __restrict__ bidx, double* __restrict__ bp,
                             int n) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) bp[r] = __ldg(b + bidx[r]);
}

void permute_in(const double* b, const int* bidx, double* bp, int n, cudaStream_t st) {
    if (n <= 0) return;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if ((reinterpret_cast<std::uintptr_t>(bp) | reinterpret_cast<std::uintptr_t>(bidx)) & 15) {  // caller's vector
        k_permute_in<<<std::min((n + 255) / 256, sms * 8), 256, 0, st>>>(b, bidx, bp, n);
        return;
    }
    const int blocks = std::max(1, std::min((n / 4 + 255) / 256, sms * 8));
    k_permute_in4<<<blocks, 256, 0, st>>>(b, bidx, bp, n);
}

// the k_wave instantiations live in wave_inst_*.cu (compiled in parallel)
void* wave_kernel_a(int width, int group, int groups, int rpl, bool trace);
void* wave_kernel_b(int width, int group, int groups, int rpl, bool trace);
void* wave_kernel_c(int width, int group, int groups, int rpl, bool trace);
void* wave_kernel_d(int width, int group, int groups, int rpl, bool trace);

void* wave_kernel(int width, int group, int groups, int rpl, bool trace) {
    for (auto f : {wave_kernel_a, wave_kernel_b, wave_kernel_c, wave_kernel_d})
        if (void* k = f(width, group, groups, rpl, trace)) return k;
    return nullptr;
}

}  // namespace hec::dev
