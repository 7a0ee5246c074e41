// Device GMRES(m): right-preconditioned, restarted, zero initial guess.
// Control flow, tolerances, lucky-breakdown / stall logic, Givens rotations and
// the reported quantities follow reference proj/src/gmres.cpp:28-137 line for
// line; the n-length work (SpMV, preconditioner, MGS, updates) runs on the GPU.
//
// Fused Krylov kernels: one MGS step = (w -= h_{i-1} v_{i-1}) + partial dot
// (w, v_i) in one pass, with a deterministic two-level reduction finished by
// the last CTA (fixed grid, fixed order: run-to-run bitwise reproducible).
// Dot products are not bitwise equal to the reference's serial ascending sum,
// so iteration counts are compared within +-1.

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cmath>
#include <vector>

#include "device_runtime.hpp"
#include "krylov.hpp"

namespace hec::dev {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    // fixed-shape tree: warp shuffles then one warp over the warp sums
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    if (warp == 0)
        for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Finishes a reduction: block partial -> partials[bid]; the last block to
// arrive sums them with a fixed-shape tree (thread t takes partials t, t+T, ..
// in order, then block_sum) into *out (optionally sqrt'ed into *out_sqrt).
// Fixed grid -> run-to-run reproducible.
__device__ __forceinline__ void finish(double part, double* partials, unsigned* counter, double* out,
                                       double* out_sqrt) {
    __shared__ double sh[32];
    __shared__ bool last;
    const double s = block_sum(part, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = s;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double t = 0.0;
        for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) t = __dadd_rn(t, __ldcg(&partials[k]));
        __syncthreads();  // sh reuse
        t = block_sum(t, sh);
        if (threadIdx.x == 0) {
            *out = t;
            if (out_sqrt) *out_sqrt = __dsqrt_rn(t);
            *counter = 0;
        }
    }
}

// w -= (*h_prev) * v_prev  (if v_prev), then *out = dot(w, v_next).
// Two elements per thread per step (16-byte loads when every vector is
// 16-byte aligned), grid-stride; memory-bound.
__global__ void __launch_bounds__(kThreads) k_mgs_step(int n, double* w, const double* v_prev, const double* h_prev,
                                                     const double* v_next, double* partials, unsigned* counter,
                                                     double* out, double* out_sqrt) {
    double acc = 0.0;
    const double h = v_prev ? *h_prev : 0.0;
    const bool self = v_next == w;
    const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(v_prev) |
                       reinterpret_cast<uintptr_t>(v_next)) & 15) == 0;
    const int stride = gridDim.x * blockDim.x;
    int i0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (vec) {
        const int n2 = n >> 1;
        double2* w2 = reinterpret_cast<double2*>(w);
        for (int i = i0; i < n2; i += stride) {
            double2 wi = w2[i];
            if (v_prev) {
                const double2 vp = __ldg(reinterpret_cast<const double2*>(v_prev) + i);
                wi.x = __dsub_rn(wi.x, __dmul_rn(h, vp.x));
                wi.y = __dsub_rn(wi.y, __dmul_rn(h, vp.y));
                w2[i] = wi;
            }
            const double2 vn = self ? wi : __ldg(reinterpret_cast<const double2*>(v_next) + i);
            acc = __dadd_rn(acc, __dmul_rn(wi.x, vn.x));
            acc = __dadd_rn(acc, __dmul_rn(wi.y, vn.y));
        }
        // an odd last element is left to the first thread of the grid
        i0 = (blockIdx.x == 0 && threadIdx.x == 0) ? 2 * n2 : n;
    }
    for (int i = i0; i < n; i += stride) {
        double wi = w[i];
        if (v_prev) {
            wi = __dsub_rn(wi, __dmul_rn(h, v_prev[i]));
            w[i] = wi;
        }
        const double vn = self ? wi : v_next[i];
        acc = __dadd_rn(acc, __dmul_rn(wi, vn));
    }
    finish(acc, partials, counter, out, out_sqrt);
}

// y = x / (*s)
__global__ void k_div(int n, double* y, const double* x, const double* s) {
    const double d = *s;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        y[i] = __ddiv_rn(x[i], d);
}

// xc = sum_i y_i v_i accumulated in i order from 0.0
__global__ void k_combine(int n, int j, double* xc, const double* V, size_t ldv, const double* y) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < j; ++i) s = __dadd_rn(s, __dmul_rn(y[i], V[i * ldv + t]));
        xc[t] = s;
    }
}

__global__ void k_add(int n, double* x, const double* d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        x[i] = __dadd_rn(x[i], d[i]);
}

__global__ void k_sqrt(const double* in, double* out) { *out = __dsqrt_rn(*in); }

}  // namespace

KrylovOps::KrylovOps(int n) : n_(n) {
    if (n < 0) throw std::invalid_argument("hec_krylov_create: negative size");
    int dev = 0, sms = 0;
    HEC_CUDA(cudaGetDevice(&dev));
    HEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid_ = std::max(1, std::min(4 * sms, (n + 2 * kThreads - 1) / (2 * kThreads)));
    HEC_CUDA(cudaMalloc(reinterpret_cast<void**>(&partials_), sizeof(double) * grid_));
    HEC_CUDA(cudaMalloc(reinterpret_cast<void**>(&counter_), sizeof(unsigned)));
    HEC_CUDA(cudaMemset(counter_, 0, sizeof(unsigned)));
}

KrylovOps::~KrylovOps() {
    cudaFree(partials_);
    cudaFree(counter_);
}

void KrylovOps::mgs(double* w, const double* v_prev, const double* h_prev, const double* v_next, double* out,
                    cudaStream_t st) {
    k_mgs_step<<<grid_, kThreads, 0, st>>>(n_, w, v_prev, h_prev, v_next, partials_, counter_, out, nullptr);
    HEC_CUDA(cudaGetLastError());
}

void KrylovOps::scale(double* y, const double* x, const double* s, cudaStream_t st) {
    k_div<<<grid_, kThreads, 0, st>>>(n_, y, x, s);
    HEC_CUDA(cudaGetLastError());
}

void KrylovOps::combine(int j, double* xc, const double* V, long long ldv, const double* y, cudaStream_t st) {
    k_combine<<<grid_, kThreads, 0, st>>>(n_, j, xc, V, static_cast<size_t>(ldv), y);
    HEC_CUDA(cudaGetLastError());
}

void KrylovOps::add(double* x, const double* d, cudaStream_t st) {
    k_add<<<grid_, kThreads, 0, st>>>(n_, x, d);
    HEC_CUDA(cudaGetLastError());
}

void KrylovOps::sqrt(const double* in, double* out, cudaStream_t st) {
    k_sqrt<<<1, 1, 0, st>>>(in, out);
    HEC_CUDA(cudaGetLastError());
}

}  // namespace hec::dev
