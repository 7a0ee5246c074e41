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

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace cg = cooperative_groups;

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
__device__ __forceinline__ double level_acc(const LevelArgs& a, int r) {
    double acc = a.b[a.b_ordered ? r : a.bidx[r]];
    for (int k = 0; k < a.width; ++k) {
        const size_t slot = static_cast<size_t>(k) * a.ld + r;
        const int d = a.ell_dep[slot];
        if (d >= 0) acc = sub_prod(acc, a.ell_val[slot], a.xs[d]);
    }
    return acc;
}

__device__ __forceinline__ void level_store(const LevelArgs& a, int r, double acc) {
    const double x = __ddiv_rn(acc, a.diag[r]);
    a.xs[a.xidx[r]] = x;
    if (a.out) {
        const int o = a.oidx[r];
        if (o >= 0) a.out[o] = x;
    }
}

// One row per thread; rows with a long remainder are left to level_row_warp
// when skip_long.
__device__ __forceinline__ void level_row(const LevelArgs& a, int r, bool skip_long) {
    const int t0 = a.tail_rp[r], t1 = a.tail_rp[r + 1];
    if (skip_long && a.long_min > 0 && t1 - t0 >= a.long_min) return;
    double acc = level_acc(a, r);
    for (int t = t0; t < t1; ++t) acc = sub_prod(acc, a.tail_val[t], a.xs[a.tail_dep[t]]);
    level_store(a, r, acc);
}

// One row per warp (the remainder loop at triangular.cpp:123-125 for long rows):
// the lanes load 32 (dep, value) pairs and gather x in parallel and form the
// products (each rounded on its own, as in sub_prod); the differences then run
// in stored order on a broadcast accumulator, so the result is the
// thread-serial one bit for bit. The next 32 entries are in flight meanwhile.
__device__ __forceinline__ void level_row_warp(const LevelArgs& a, int r, int lane) {
    const int t0 = a.tail_rp[r], t1 = a.tail_rp[r + 1];
    double acc = level_acc(a, r);  // every lane the same (broadcast loads)
    auto prod = [&](int t) { return t < t1 ? __dmul_rn(a.tail_val[t], a.xs[a.tail_dep[t]]) : 0.0; };
    double p = prod(t0 + lane);
    for (int t = t0; t < t1; t += 32) {
        const double pn = prod(t + 32 + lane);
        const int m = min(32, t1 - t);
        for (int q = 0; q < m; ++q) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, p, q));
        p = pn;
    }
    if (lane == 0) level_store(a, r, acc);
}

// blocks [0, row_blocks) take the level's rows a thread each, the blocks after
// them its long rows [l0, l1) a warp each.
__global__ void k_level_rows(const LevelArgs* __restrict__ pa, int r0, int r1, int l0, int l1, int row_blocks) {
    const LevelArgs& a = *pa;
    if (static_cast<int>(blockIdx.x) < row_blocks) {
        const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
        if (r < r1) level_row(a, r, true);
        return;
    }
    const int w = l0 + ((blockIdx.x - row_blocks) * blockDim.x + threadIdx.x) / 32;
    if (w < l1) level_row_warp(a, a.long_rows[w], threadIdx.x & 31);
}

// All levels in one cooperative launch, a grid-wide barrier between them (the
// reference's per-level barrier, triangular.cpp:128, as a grid barrier instead of
// a kernel boundary): the measured alternative to the per-level launches.
__global__ void __launch_bounds__(256) k_level_persist(const LevelArgs* __restrict__ pa,
                                                       const int* __restrict__ level_starts, int nlev) {
    cg::grid_group grid = cg::this_grid();
    const LevelArgs& a = *pa;
    const int stride = gridDim.x * blockDim.x;
    for (int k = 0; k < nlev; ++k) {
        const int r1 = level_starts[k + 1];
        for (int r = level_starts[k] + blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += stride)
            level_row(a, r, false);
        if (k + 1 < nlev) grid.sync();
    }
}

void launch_levels_persist(const LevelArgs* dev_args, const int* level_starts_dev, int nlev, cudaStream_t st) {
    static int blocks = 0;
    if (!blocks) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_level_persist, 256, 0);
        blocks = std::max(1, sms * std::max(1, per));
    }
    void* args[] = {const_cast<LevelArgs**>(&dev_args), const_cast<int**>(&level_starts_dev), &nlev};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(&k_level_persist), dim3(blocks), dim3(256), args, 0, st);
}

__global__ void k_set_level_args(LevelArgs a, LevelArgs* dst) { *dst = a; }

void set_level_args(const LevelArgs& a, LevelArgs* dev, cudaStream_t st) {
    k_set_level_args<<<1, 1, 0, st>>>(a, dev);
}

void launch_levels(const LevelArgs* dev_args, const int* level_starts_host, const int* long_starts_host, int nlev,
                   cudaStream_t st) {
    for (int k = 0; k < nlev; ++k) {
        const int r0 = level_starts_host[k], r1 = level_starts_host[k + 1];
        const int l0 = long_starts_host[k], l1 = long_starts_host[k + 1];
        const int m = r1 - r0;
        const int tpb = m >= 256 ? 256 : (m >= 128 ? 128 : 64);
        const int row_blocks = (m + tpb - 1) / tpb;
        const int long_blocks = ((l1 - l0) * 32 + tpb - 1) / tpb;
        k_level_rows<<<row_blocks + long_blocks, tpb, 0, st>>>(dev_args, r0, r1, l0, l1, row_blocks);
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

// bp[wpos[o]] = b[o]: the inverse of the gather above, for a slice of the input
// that has just arrived (coalesced reads, one scattered store per row)
__global__ void __launch_bounds__(256) k_scatter_rows(const double* __restrict__ b, const int* __restrict__ wpos,
                                                      double* __restrict__ bp, int n) {
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) bp[__ldcs(wpos + o)] = __ldcs(b + o);
}

void scatter_rows(const double* b, const int* wpos, double* bp, int n, cudaStream_t st) {
    if (n <= 0) return;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    k_scatter_rows<<<std::min((n + 255) / 256, sms * 8), 256, 0, st>>>(b, wpos, bp, n);
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
