#pragma once
// Device GMRES(m) entry point (see krylov.cu).

#include <cuda_runtime.h>

#include <vector>

#include "gmres_engine.hpp"

namespace hec::dev {

class DeviceSpmv;
class DevicePrecond;

// The fused Krylov vector kernels of gmres_device, for drivers that add their
// own reductions across GPUs (the RAS layer). All results stay on the device;
// dots use a fixed-shape two-level reduction (run-to-run reproducible).
class KrylovOps {
public:
    explicit KrylovOps(int n);
    ~KrylovOps();
    KrylovOps(const KrylovOps&) = delete;
    KrylovOps& operator=(const KrylovOps&) = delete;
    int n() const { return n_; }
    // w -= (*h_prev) v_prev (if v_prev), then *out = dot(w, v_next) (v_next may be w)
    void mgs(double* w, const double* v_prev, const double* h_prev, const double* v_next, double* out,
             cudaStream_t st);
    void scale(double* y, const double* x, const double* s, cudaStream_t st);   // y = x / *s
    void combine(int j, double* xc, const double* V, long long ldv, const double* y, cudaStream_t st);  // sum y_i V_i
    void add(double* x, const double* d, cudaStream_t st);                       // x += d
    void sqrt(const double* in, double* out, cudaStream_t st);                   // *out = sqrt(*in)

private:
    int n_ = 0, grid_ = 1;
    double* partials_ = nullptr;
    unsigned* counter_ = nullptr;
};

}  // namespace hec::dev
