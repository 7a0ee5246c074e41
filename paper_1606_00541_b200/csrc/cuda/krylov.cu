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

GmresOutcome gmres_device(const DeviceSpmv& A, DevicePrecond* M, const double* b_host, const GmresParams& cfg,
                          double* x_host) {
    if (A.n_rows() != A.n_cols()) throw std::invalid_argument("gmres: matrix must be square");
    if (cfg.restart < 1) throw std::invalid_argument("gmres: restart must be >= 1");
    if (cfg.max_iters < 0) throw std::invalid_argument("gmres: max_iters must be >= 0");
    if (cfg.rel_tol < 0.0 || cfg.abs_tol < 0.0) throw std::invalid_argument("gmres: tolerances must be >= 0");
    if (M && M->n() != A.n_rows()) throw std::invalid_argument("gmres: preconditioner size mismatch");

    const auto t0 = std::chrono::steady_clock::now();
    const int n = A.n_rows();
    const int mr = cfg.restart;
    GmresOutcome out;
    cudaStream_t st = nullptr;
    HEC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } guard{st};

    int dev = 0, sms = 0;
    HEC_CUDA(cudaGetDevice(&dev));
    HEC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::max(1, std::min(4 * sms, (n + 2 * kThreads - 1) / (2 * kThreads)));
    const size_t ldv = static_cast<size_t>((std::max(n, 1) + 3) / 4 * 4);  // 32-byte aligned basis columns

    DevBuf<double> V((mr + 1) * ldv), w(ldv), z(ldv), r(ldv), x(ldv), b(ldv), yv(mr + 1);
    DevBuf<double> hcol(mr + 3), partials(grid), scal(2);
    DevBuf<unsigned> counter(1);
    HEC_CUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned), st));
    HEC_CUDA(cudaMemcpyAsync(b.p, b_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    HEC_CUDA(cudaMemsetAsync(x.p, 0, sizeof(double) * ldv, st));
    out.launches += 0;

    auto dot_into = [&](const double* a, double* dst, double* dst_sqrt) {
        // dot(a, a) via the fused kernel with no axpy part
        k_mgs_step<<<grid, kThreads, 0, st>>>(n, const_cast<double*>(a), nullptr, nullptr, a, partials.p,
                                                counter.p, dst, dst_sqrt);
        ++out.launches;
    };
    auto fetch = [&](const double* src, double* dst, int count) {
        HEC_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
        HEC_CUDA(cudaStreamSynchronize(st));
    };

    double bn[2];
    dot_into(b.p, scal.p, scal.p + 1);
    fetch(scal.p, bn, 2);
    const double bnorm = bn[1];
    const double threshold = std::max(cfg.rel_tol * bnorm, cfg.abs_tol);

    std::vector<double> h(static_cast<size_t>(mr + 1) * mr, 0.0), cs(mr), sn(mr), g(mr + 1), y(mr);
    HEC_CUDA(cudaMemcpyAsync(r.p, b.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    double rnorm = bnorm;
    bool stalled = false;
    double* rnorm_dev = scal.p + 1;  // holds ||r|| on the device

    while (true) {
        if (rnorm <= threshold) {
            out.converged = true;
            break;
        }
        if (out.iterations >= cfg.max_iters || stalled) break;
        k_div<<<grid, kThreads, 0, st>>>(n, V.p, r.p, rnorm_dev);
        ++out.launches;
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = rnorm;

        int j = 0;
        bool lucky = false;
        while (j < mr && out.iterations < cfg.max_iters) {
            double* vj = V.p + j * ldv;
            if (M) {
                M->apply(vj, z.p, st);
                out.launches += M->lower().launches_per_solve() + M->upper().launches_per_solve();
                A.run(z.p, w.p, st);
            } else {
                A.run(vj, w.p, st);
            }
            ++out.launches;
            // MGS: step i computes h_ij after removing the (i-1) component
            for (int i = 0; i <= j; ++i) {
                k_mgs_step<<<grid, kThreads, 0, st>>>(n, w.p, i ? V.p + (i - 1) * ldv : nullptr,
                                                       i ? hcol.p + (i - 1) : nullptr, V.p + i * ldv,
                                                       partials.p, counter.p, hcol.p + i, nullptr);
                ++out.launches;
            }
            // last removal fused with ||w||^2, then v_{j+1} = w / ||w||
            k_mgs_step<<<grid, kThreads, 0, st>>>(n, w.p, vj, hcol.p + j, w.p, partials.p, counter.p,
                                                   hcol.p + j + 2, hcol.p + j + 1);
            ++out.launches;
            k_div<<<grid, kThreads, 0, st>>>(n, V.p + (j + 1) * ldv, w.p, hcol.p + j + 1);
            ++out.launches;
            std::vector<double> hc(j + 2);
            fetch(hcol.p, hc.data(), j + 2);
            for (int i = 0; i <= j; ++i) h[i + j * (mr + 1)] = hc[i];
            const double hjj1 = hc[j + 1];
            h[(j + 1) + j * (mr + 1)] = hjj1;
            if (!(hjj1 > 1e-300)) lucky = true;

            for (int i = 0; i < j; ++i) {
                const double hi = h[i + j * (mr + 1)];
                const double hi1 = h[(i + 1) + j * (mr + 1)];
                h[i + j * (mr + 1)] = cs[i] * hi + sn[i] * hi1;
                h[(i + 1) + j * (mr + 1)] = -sn[i] * hi + cs[i] * hi1;
            }
            const double hjj = h[j + j * (mr + 1)];
            const double denom = std::hypot(hjj, hjj1);
            if (denom > 0.0) {
                cs[j] = hjj / denom;
                sn[j] = hjj1 / denom;
            } else {
                cs[j] = 1.0;
                sn[j] = 0.0;
            }
            h[j + j * (mr + 1)] = denom;
            h[(j + 1) + j * (mr + 1)] = 0.0;
            const double gj = g[j];
            g[j] = cs[j] * gj;
            g[j + 1] = -sn[j] * gj;

            ++out.iterations;
            ++j;
            const double est = std::fabs(g[j]);
            out.inner_residuals.push_back(est);
            if (est <= threshold || lucky) break;
        }

        for (int i = j - 1; i >= 0; --i) {
            double s = g[i];
            for (int t = i + 1; t < j; ++t) s -= h[i + t * (mr + 1)] * y[t];
            y[i] = s / h[i + i * (mr + 1)];
        }
        HEC_CUDA(cudaMemcpyAsync(yv.p, y.data(), sizeof(double) * std::max(j, 1), cudaMemcpyHostToDevice, st));
        k_combine<<<grid, kThreads, 0, st>>>(n, j, w.p, V.p, ldv, yv.p);
        ++out.launches;
        if (M) {
            M->apply(w.p, z.p, st);
            out.launches += M->lower().launches_per_solve() + M->upper().launches_per_solve();
            k_add<<<grid, kThreads, 0, st>>>(n, x.p, z.p);
        } else {
            k_add<<<grid, kThreads, 0, st>>>(n, x.p, w.p);
        }
        ++out.launches;
        A.residual(b.p, x.p, r.p, st);
        ++out.launches;
        dot_into(r.p, scal.p, rnorm_dev);
        double rr[2];
        fetch(scal.p, rr, 2);
        const double rn = rr[1];
        if (lucky && rn > threshold) stalled = true;
        rnorm = rn;
    }
    out.final_relative_residual = bnorm > 0.0 ? rnorm / bnorm : rnorm;
    HEC_CUDA(cudaMemcpyAsync(x_host, x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    HEC_CUDA(cudaStreamSynchronize(st));
    HEC_CUDA(cudaGetLastError());
    out.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

}  // namespace hec::dev
