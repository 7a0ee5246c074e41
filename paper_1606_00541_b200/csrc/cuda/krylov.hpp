#pragma once
// Device GMRES(m) entry point (see krylov.cu).

#include <vector>

namespace hec::dev {

class DeviceSpmv;
class DevicePrecond;

struct GmresParams {
    int restart = 20;
    int max_iters = 10000;
    double rel_tol = 1e-6;
    double abs_tol = 0.0;
};

struct GmresOutcome {
    bool converged = false;
    int iterations = 0;
    double final_relative_residual = 0.0;
    double solve_seconds = 0.0;
    long long launches = 0;
    std::vector<double> inner_residuals;
};

GmresOutcome gmres_device(const DeviceSpmv& A, DevicePrecond* M, const double* b_host, const GmresParams& cfg,
                          double* x_host);

}  // namespace hec::dev
