#pragma once
// Device GMRES(m) engine (gmres_engine.cu): one GPU, or one RAS subdomain per
// rank with halo exchanges and dot all-reduces through a Comm.

#include <cuda_runtime.h>

#include <vector>

namespace hec::dev {

class DeviceSpmv;
class DevicePrecond;
class Comm;

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
    long long allreduces = 0, exchanges = 0;
    std::vector<double> inner_residuals;
};

// The local part of a distributed operator. Vectors are [own | halo] of n_loc
// entries; the solution and right-hand side are the owned n_own rows.
struct DistSystem {
    int n_own = 0, n_loc = 0;
    const DeviceSpmv* A = nullptr;  // owned rows, columns in [own | halo]
    DevicePrecond* M = nullptr;     // local form: input n_loc, output n_own (or nullptr)
    const int* send_idx = nullptr;  // device, own positions to send (peer order)
    int n_send = 0;
    std::vector<int> send_off, recv_off;  // [world + 1]
    Comm* comm = nullptr;                 // nullptr = one rank
};

// Fills vloc[n_own ..) (the halo) from the owning ranks: pack the rows peers
// need into sendbuf (n_send doubles), then the Comm's exchange. Collective.
void halo_exchange(const DistSystem& S, double* vloc, double* sendbuf, cudaStream_t st);

// b_own / x_own: device pointers of n_own doubles; enqueued on st, synchronous.
GmresOutcome gmres_dist(DistSystem& S, const double* b_own, double* x_own, const GmresParams& cfg, cudaStream_t st);

// Single GPU with host vectors (hec::gmres, hec_gmres_solve).
GmresOutcome gmres_device(const DeviceSpmv& A, DevicePrecond* M, const double* b_host, const GmresParams& cfg,
                          double* x_host);

}  // namespace hec::dev
