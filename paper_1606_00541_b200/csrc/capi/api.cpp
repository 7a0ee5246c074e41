// The two public faces of the library:
//  * the drop-in C++ API (hec::solve / hec::apply / hec::gmres) whose host
//    setup lives in csrc/host and whose per-iteration work runs on the B200;
//  * the C-ABI of include/hecsolve_c.h (status codes, opaque handles).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../cuda/comm.hpp"
#include "../cuda/device_runtime.hpp"
#include "../cuda/krylov.hpp"
#include "../host/ras_plan.hpp"
#include "hecsolve/device.hpp"
#include "hecsolve/errors.hpp"
#include "hecsolve/gmres.hpp"
#include "hecsolve/ilu.hpp"
#include "hecsolve/poisson.hpp"
#include "hecsolve/precond.hpp"
#include "hecsolve/triangular.hpp"
#include "hecsolve_c.h"

struct hec_tri {
    std::unique_ptr<hec::dev::DeviceTri> impl;
};
struct hec_precond {
    std::unique_ptr<hec::dev::DevicePrecond> impl;
};
struct hec_spmv {
    std::unique_ptr<hec::dev::DeviceSpmv> impl;
};
struct hec_csr {
    hec::CsrMatrix m;
};
struct hec_prep {
    std::shared_ptr<const hec::PreparedTriangular> p;
};
struct hec_bp {
    hec::BlockPreconditioner m;
    hec_prep l, u;
};
struct hec_krylov {
    std::unique_ptr<hec::dev::KrylovOps> impl;
};
struct hec_hec {
    hec::HecMatrix m;
};
struct hec_ras_plan {
    hec::ras::Plan plan;
};
struct hec_ras {
    hec_ras_plan p;
    std::unique_ptr<hec::dev::Comm> comm;
    std::unique_ptr<hec::dev::DevicePrecond> M;
    std::unique_ptr<hec::dev::DeviceSpmv> A;
    hec::dev::DevBuf<int> send_idx;
    hec::dev::DevBuf<double> vloc, sendbuf, h_r, h_z;
    cudaStream_t stream = nullptr;
    long long allreduces = 0, exchanges = 0, launches = 0;
    ~hec_ras() {
        if (stream) cudaStreamDestroy(stream);
    }
};
struct hec_partition {
    int n = 0, parts = 0;
    std::vector<int> part_of, ext_offsets, ext_rows;
};

namespace hec {

// ------------------------------------------------------------ options ----
namespace device {
namespace {
std::atomic<int> g_strategy{HEC_STRATEGY_AUTO}, g_ctas{0}, g_threads{0};
}
void set_options(const Options& o) {
    g_strategy = o.strategy;
    g_ctas = o.ctas;
    g_threads = o.threads;
}
Options options() { return Options{g_strategy.load(), g_ctas.load(), g_threads.load()}; }

TriMirror::~TriMirror() { delete handle; }
PrecondMirror::~PrecondMirror() { delete handle; }
}  // namespace device

namespace {

dev::TriOptions tri_options(const hec_tri_options* o) {
    dev::TriOptions t;
    const device::Options d = device::options();
    t.strategy = o ? o->strategy : d.strategy;
    t.ctas = o ? o->ctas : d.ctas;
    t.threads = o ? o->threads : d.threads;
    return t;
}

plan::TriSource source_of(const PreparedTriangular& p) {
    plan::TriSource s;
    s.n = p.n;
    s.reversed = p.reversal_applied;
    s.nlev = p.schedule.nlev;
    s.level_starts = p.schedule.level_starts.data();
    s.inv_perm = p.schedule.inv_perm.data();
    s.ell_width = p.hec.ell.width;
    s.ell_cols = p.hec.ell.col_indices.data();
    s.ell_vals = p.hec.ell.values.data();
    s.csr_rp = p.hec.csr.row_offsets.data();
    s.csr_cols = p.hec.csr.col_indices.data();
    s.csr_vals = p.hec.csr.values.data();
    if (static_cast<int>(p.schedule.inv_perm.size()) != p.n ||
        static_cast<int>(p.schedule.level_starts.size()) != p.schedule.nlev + 1 ||
        static_cast<int>(p.hec.csr.row_offsets.size()) != p.n + 1 ||
        p.hec.ell.col_indices.size() != static_cast<std::size_t>(p.hec.ell.width) * p.n)
        throw std::invalid_argument("solve: inconsistent PreparedTriangular");
    return s;
}

hec_tri* build_tri(const PreparedTriangular& p) {
    auto h = std::make_unique<hec_tri>();
    h->impl = std::make_unique<dev::DeviceTri>(source_of(p), tri_options(nullptr));
    return h.release();
}

hec_precond* build_precond(const BlockPreconditioner& m) {
    const int s = m.partition.n_parts;
    const int n_ext = m.offsets.empty() ? 0 : m.offsets[s];
    std::vector<int> gather(n_ext);
    std::vector<char> owned(n_ext);
    for (int p = 0; p < s; ++p)
        for (std::size_t li = 0; li < m.extended_parts[p].size(); ++li) {
            gather[m.offsets[p] + li] = m.extended_parts[p][li];
            owned[m.offsets[p] + li] = m.restriction[p][li];
        }
    auto h = std::make_unique<hec_precond>();
    h->impl = std::make_unique<dev::DevicePrecond>(m.n, n_ext, gather.data(), owned.data(),
                                                   source_of(m.prepared_l), source_of(m.prepared_u),
                                                   tri_options(nullptr));
    return h.release();
}

}  // namespace

// The device mirror is built on first use and shared by copies of the object
// (the reference's objects are immutable after construction, SPEC.md). A copy
// owns separate arrays: it is recognised by their addresses and gets a device
// copy of its own instead of the original's (returns nullptr: build one-off).
hec_tri_t device_handle(const PreparedTriangular& p) {
    if (!p.device) throw std::invalid_argument("solve: PreparedTriangular has no device slot (use prepare_*)");
    std::lock_guard<std::mutex> g(p.device->mu);
    const void* src = p.hec.csr.values.data();
    if (!p.device->handle) {
        p.device->handle = build_tri(p);
        p.device->source = src;
    }
    return p.device->source == src ? p.device->handle : nullptr;
}

hec_precond_t device_handle(const BlockPreconditioner& m) {
    if (!m.device) throw std::invalid_argument("apply: BlockPreconditioner has no device slot");
    std::lock_guard<std::mutex> g(m.device->mu);
    const void* src = m.prepared_l.hec.csr.values.data();
    if (!m.device->handle) {
        m.device->handle = build_precond(m);
        m.device->source = src;
    }
    return m.device->source == src ? m.device->handle : nullptr;
}

// ------------------------------------------------------ drop-in C++ API ----
std::vector<double> solve(const PreparedTriangular& p, const std::vector<double>& b, int /*workers*/) {
    if (static_cast<int>(b.size()) != p.n) throw std::invalid_argument("solve: dimension mismatch");
    std::vector<double> x(p.n);
    if (p.n == 0) return x;
    if (hec_tri_t h = p.device ? device_handle(p) : nullptr) {
        h->impl->solve_host(b.data(), x.data());
    } else {  // hand-assembled object or a copy: build a one-off device copy
        std::unique_ptr<hec_tri> t(build_tri(p));
        t->impl->solve_host(b.data(), x.data());
    }
    return x;
}

std::vector<double> apply(const BlockPreconditioner& m, const std::vector<double>& r, int /*workers*/) {
    if (static_cast<int>(r.size()) != m.n) throw std::invalid_argument("apply: dimension mismatch");
    std::vector<double> x(m.n);
    if (m.n == 0) return x;
    if (hec_precond_t h = m.device ? device_handle(m) : nullptr) {
        h->impl->apply_host(r.data(), x.data());
    } else {  // hand-assembled object or a copy: one-off device copy
        std::unique_ptr<hec_precond> d(build_precond(m));
        d->impl->apply_host(r.data(), x.data());
    }
    return x;
}

SolveResult gmres(const CsrMatrix& a, const std::vector<double>& b, const BlockPreconditioner* m,
                  const SolverConfig& cfg, int /*workers*/) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("gmres: matrix must be square");
    if (static_cast<int>(b.size()) != a.n_rows) throw std::invalid_argument("gmres: dimension mismatch");
    if (cfg.restart < 1) throw std::invalid_argument("gmres: restart must be >= 1");
    if (cfg.max_iters < 0) throw std::invalid_argument("gmres: max_iters must be >= 0");
    if (cfg.rel_tol < 0.0 || cfg.abs_tol < 0.0) throw std::invalid_argument("gmres: tolerances must be >= 0");
    if (m && m->n != a.n_rows) throw std::invalid_argument("gmres: preconditioner size mismatch");
    dev::DeviceSpmv A(a.n_rows, a.n_cols, a.row_offsets.data(), a.col_indices.data(), a.values.data());
    std::unique_ptr<hec_precond> tmp;
    dev::DevicePrecond* M = nullptr;
    if (m) {
        if (hec_precond_t h = m->device ? device_handle(*m) : nullptr) {
            M = h->impl.get();
        } else {
            tmp.reset(build_precond(*m));
            M = tmp->impl.get();
        }
    }
    dev::GmresParams gp{cfg.restart, cfg.max_iters, cfg.rel_tol, cfg.abs_tol};
    SolveResult res;
    res.x.assign(a.n_rows, 0.0);
    dev::GmresOutcome o = dev::gmres_device(A, M, b.data(), gp, res.x.data());
    res.report.converged = o.converged;
    res.report.iterations = o.iterations;
    res.report.final_relative_residual = o.final_relative_residual;
    res.report.solve_seconds = o.solve_seconds;
    res.report.inner_residuals = std::move(o.inner_residuals);
    return res;
}

}  // namespace hec

// =========================================================== C-ABI ========
namespace {

thread_local std::string t_msg;
thread_local int t_row = -1, t_block = -1;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return HEC_OK;
    } catch (const hec::ZeroPivotError& e) {
        t_msg = e.what();
        t_row = e.row();
        t_block = e.block();
        return HEC_EZEROPIVOT;
    } catch (const std::invalid_argument& e) {
        t_msg = e.what();
        return HEC_EINVAL;
    } catch (const std::out_of_range& e) {
        t_msg = e.what();
        return HEC_ERANGE;
    } catch (const std::overflow_error& e) {
        t_msg = e.what();
        return HEC_EOVERFLOW;
    } catch (const std::bad_alloc& e) {
        t_msg = std::string("out of memory: ") + e.what();
        return HEC_ERUNTIME;
    } catch (const std::exception& e) {
        t_msg = e.what();
        return HEC_ERUNTIME;
    } catch (...) {
        t_msg = "unknown error";
        return HEC_ERUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string(what) + ": null argument");
}

hec::plan::TriSource raw_source(int n, int rev, int nlev, const int* ls, const int* ip, int w, const int* ec,
                                const double* ev, const int* rp, const int* cc, const double* cv) {
    hec::plan::TriSource s;
    s.n = n;
    s.reversed = rev != 0;
    s.nlev = nlev;
    s.level_starts = ls;
    s.inv_perm = ip;
    s.ell_width = w;
    s.ell_cols = ec;
    s.ell_vals = ev;
    s.csr_rp = rp;
    s.csr_cols = cc;
    s.csr_vals = cv;
    return s;
}

void fill_info(const hec::dev::TriStats& s, hec_tri_info* info) {
    info->n = s.n;
    info->nlev = s.nlev;
    info->strategy = s.strategy;
    info->ctas = s.ctas;
    info->threads = s.threads;
    info->chunks = s.chunks;
    info->nnz = s.nnz;
    info->device_bytes = s.device_bytes;
    info->alg_bytes = s.alg_bytes;
    info->predicted_us = s.predicted_us;
    info->layout = s.layout;
    info->group = s.group;
    info->groups = s.groups;
    info->rows_per_lane = s.rpl;
    info->width = s.width;
    info->ring = s.ring;
    info->halo_ring = s.halo_ring;
    info->inflight = s.slots;
    info->wave_len = s.wave_len;
}

hec::WidthPolicy policy_of(int mode, int width) {
    return mode == 1 ? hec::WidthPolicy::fixed(width) : hec::WidthPolicy::automatic();
}

}  // namespace

extern "C" {

const char* hec_last_error(void) { return t_msg.c_str(); }
int hec_last_error_row(void) { return t_row; }
int hec_last_error_block(void) { return t_block; }
const char* hec_version(void) { return "hecsolve-b200 0.1.0 sm_100a"; }

int hec_device_available(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count > 0 ? 1 : 0;
}

// ---- device path ----
int hec_tri_create(int n, int reversal_applied, int nlev, const int* level_starts, const int* inv_perm,
                   int ell_width, const int* ell_cols, const double* ell_vals, const int* csr_row_offsets,
                   const int* csr_cols, const double* csr_vals, const hec_tri_options* options, hec_tri_t* out) {
    return guarded([&] {
        need(out, "hec_tri_create");
        auto h = std::make_unique<hec_tri>();
        h->impl = std::make_unique<hec::dev::DeviceTri>(
            raw_source(n, reversal_applied, nlev, level_starts, inv_perm, ell_width, ell_cols, ell_vals,
                       csr_row_offsets, csr_cols, csr_vals),
            hec::tri_options(options));
        *out = h.release();
    });
}

int hec_tri_solve(hec_tri_t t, const double* b_dev, double* x_dev, void* stream) {
    return guarded([&] {
        need(t, "hec_tri_solve");
        if (t->impl->n() > 0 && (!b_dev || !x_dev)) throw std::invalid_argument("hec_tri_solve: null vector");
        if (b_dev == x_dev && t->impl->n() > 0) throw std::invalid_argument("hec_tri_solve: b and x must not alias");
        t->impl->solve(b_dev, x_dev, nullptr, static_cast<cudaStream_t>(stream));
    });
}

int hec_tri_permute_in(hec_tri_t t, const double* b_dev, double* bp_dev, void* stream) {
    return guarded([&] {
        need(t, "hec_tri_permute_in");
        if (t->impl->n() > 0 && (!b_dev || !bp_dev)) throw std::invalid_argument("hec_tri_permute_in: null vector");
        if (reinterpret_cast<std::uintptr_t>(bp_dev) & 15)
            throw std::invalid_argument("hec_tri_permute_in: bp must be 16-byte aligned");
        t->impl->permute(b_dev, bp_dev, static_cast<cudaStream_t>(stream));
    });
}

int hec_tri_solve_ordered(hec_tri_t t, const double* bp_dev, double* x_dev, void* stream) {
    return guarded([&] {
        need(t, "hec_tri_solve_ordered");
        if (t->impl->n() > 0 && (!bp_dev || !x_dev)) throw std::invalid_argument("hec_tri_solve_ordered: null vector");
        if (bp_dev == x_dev && t->impl->n() > 0)
            throw std::invalid_argument("hec_tri_solve_ordered: bp and x must not alias");
        if (reinterpret_cast<std::uintptr_t>(bp_dev) & 15)
            throw std::invalid_argument("hec_tri_solve_ordered: bp must be 16-byte aligned");
        t->impl->solve_ordered(bp_dev, x_dev, nullptr, static_cast<cudaStream_t>(stream));
    });
}

int hec_tri_solve_wave(hec_tri_t t, const double* bp_dev, double* xw_dev, void* stream) {
    return guarded([&] {
        need(t, "hec_tri_solve_wave");
        if (t->impl->n() > 0 && (!bp_dev || !xw_dev)) throw std::invalid_argument("hec_tri_solve_wave: null vector");
        if (bp_dev == xw_dev && t->impl->n() > 0)
            throw std::invalid_argument("hec_tri_solve_wave: bp and xw must not alias");
        if (reinterpret_cast<std::uintptr_t>(bp_dev) & 15)
            throw std::invalid_argument("hec_tri_solve_wave: bp must be 16-byte aligned");
        t->impl->solve_wave(bp_dev, xw_dev, nullptr, static_cast<cudaStream_t>(stream));
    });
}

int hec_tri_permute_out(hec_tri_t t, const double* xw_dev, double* x_dev, void* stream) {
    return guarded([&] {
        need(t, "hec_tri_permute_out");
        if (t->impl->n() > 0 && (!xw_dev || !x_dev)) throw std::invalid_argument("hec_tri_permute_out: null vector");
        if (xw_dev == x_dev && t->impl->n() > 0)
            throw std::invalid_argument("hec_tri_permute_out: xw and x must not alias");
        t->impl->permute_out(xw_dev, x_dev, static_cast<cudaStream_t>(stream));
    });
}

int hec_tri_solve_traced(hec_tri_t t, const double* b_dev, double* x_dev, void* stream,
                         unsigned long long* trace_dev, int* cta_chunk0) {
    return guarded([&] {
        need(t, "hec_tri_solve_traced");
        if (cta_chunk0) {
            const auto& v = t->impl->cta_chunk0();
            std::copy(v.begin(), v.end(), cta_chunk0);
        }
        if (b_dev && x_dev) t->impl->solve(b_dev, x_dev, nullptr, static_cast<cudaStream_t>(stream), trace_dev);
    });
}

int hec_tri_solve_host(hec_tri_t t, const double* b, double* x) {
    return guarded([&] {
        need(t, "hec_tri_solve_host");
        t->impl->solve_host(b, x);
    });
}

int hec_tri_query(hec_tri_t t, hec_tri_info* info) {
    return guarded([&] {
        need(t, "hec_tri_query");
        need(info, "hec_tri_query");
        fill_info(t->impl->stats(), info);
    });
}

int hec_tri_destroy(hec_tri_t t) {
    return guarded([&] { delete t; });
}

int hec_precond_create(int n, int n_ext, const int* gather, const char* owned, int l_nlev,
                       const int* l_level_starts, const int* l_inv_perm, int l_ell_width, const int* l_ell_cols,
                       const double* l_ell_vals, const int* l_csr_row_offsets, const int* l_csr_cols,
                       const double* l_csr_vals, int u_nlev, const int* u_level_starts, const int* u_inv_perm,
                       int u_ell_width, const int* u_ell_cols, const double* u_ell_vals,
                       const int* u_csr_row_offsets, const int* u_csr_cols, const double* u_csr_vals,
                       const hec_tri_options* options, hec_precond_t* out) {
    return guarded([&] {
        need(out, "hec_precond_create");
        if (gather) need(owned, "hec_precond_create");
        auto h = std::make_unique<hec_precond>();
        h->impl = std::make_unique<hec::dev::DevicePrecond>(
            n, n_ext, gather, owned,
            raw_source(n_ext, 0, l_nlev, l_level_starts, l_inv_perm, l_ell_width, l_ell_cols, l_ell_vals,
                       l_csr_row_offsets, l_csr_cols, l_csr_vals),
            raw_source(n_ext, 1, u_nlev, u_level_starts, u_inv_perm, u_ell_width, u_ell_cols, u_ell_vals,
                       u_csr_row_offsets, u_csr_cols, u_csr_vals),
            hec::tri_options(options));
        *out = h.release();
    });
}

int hec_precond_create_local(int n_in, int n_out, int n_ext, const int* gather, const int* out_index, int l_nlev,
                             const int* l_level_starts, const int* l_inv_perm, int l_ell_width, const int* l_ell_cols,
                             const double* l_ell_vals, const int* l_csr_row_offsets, const int* l_csr_cols,
                             const double* l_csr_vals, int u_nlev, const int* u_level_starts, const int* u_inv_perm,
                             int u_ell_width, const int* u_ell_cols, const double* u_ell_vals,
                             const int* u_csr_row_offsets, const int* u_csr_cols, const double* u_csr_vals,
                             const hec_tri_options* options, hec_precond_t* out) {
    return guarded([&] {
        need(out, "hec_precond_create_local");
        auto h = std::make_unique<hec_precond>();
        h->impl = std::make_unique<hec::dev::DevicePrecond>(
            n_in, n_out, n_ext, gather, out_index,
            raw_source(n_ext, 0, l_nlev, l_level_starts, l_inv_perm, l_ell_width, l_ell_cols, l_ell_vals,
                       l_csr_row_offsets, l_csr_cols, l_csr_vals),
            raw_source(n_ext, 1, u_nlev, u_level_starts, u_inv_perm, u_ell_width, u_ell_cols, u_ell_vals,
                       u_csr_row_offsets, u_csr_cols, u_csr_vals),
            hec::tri_options(options));
        *out = h.release();
    });
}

int hec_krylov_create(int n, hec_krylov_t* out) {
    return guarded([&] {
        need(out, "hec_krylov_create");
        hec::dev::require_device();
        auto h = std::make_unique<hec_krylov>();
        h->impl = std::make_unique<hec::dev::KrylovOps>(n);
        *out = h.release();
    });
}
int hec_krylov_mgs(hec_krylov_t k, double* w, const double* v_prev, const double* h_prev, const double* v_next,
                   double* out, void* stream) {
    return guarded([&] {
        need(k, "hec_krylov_mgs");
        if (v_prev && !h_prev) throw std::invalid_argument("hec_krylov_mgs: v_prev needs h_prev");
        k->impl->mgs(w, v_prev, h_prev, v_next, out, static_cast<cudaStream_t>(stream));
    });
}
int hec_krylov_scale(hec_krylov_t k, double* y, const double* x, const double* s, void* stream) {
    return guarded([&] {
        need(k, "hec_krylov_scale");
        k->impl->scale(y, x, s, static_cast<cudaStream_t>(stream));
    });
}
int hec_krylov_combine(hec_krylov_t k, int j, double* xc, const double* V, long long ldv, const double* y,
                       void* stream) {
    return guarded([&] {
        need(k, "hec_krylov_combine");
        k->impl->combine(j, xc, V, ldv, y, static_cast<cudaStream_t>(stream));
    });
}
int hec_krylov_add(hec_krylov_t k, double* x, const double* d, void* stream) {
    return guarded([&] {
        need(k, "hec_krylov_add");
        k->impl->add(x, d, static_cast<cudaStream_t>(stream));
    });
}
int hec_krylov_sqrt(hec_krylov_t k, const double* in, double* out, void* stream) {
    return guarded([&] {
        need(k, "hec_krylov_sqrt");
        k->impl->sqrt(in, out, static_cast<cudaStream_t>(stream));
    });
}
int hec_krylov_destroy(hec_krylov_t k) {
    return guarded([&] { delete k; });
}

int hec_precond_apply(hec_precond_t m, const double* r_dev, double* x_dev, void* stream) {
    return guarded([&] {
        need(m, "hec_precond_apply");
        m->impl->apply(r_dev, x_dev, static_cast<cudaStream_t>(stream));
    });
}

int hec_precond_apply_host(hec_precond_t m, const double* r, double* x) {
    return guarded([&] {
        need(m, "hec_precond_apply_host");
        m->impl->apply_host(r, x);
    });
}

int hec_precond_query(hec_precond_t m, hec_tri_info* l_info, hec_tri_info* u_info) {
    return guarded([&] {
        need(m, "hec_precond_query");
        if (l_info) fill_info(m->impl->lower().stats(), l_info);
        if (u_info) fill_info(m->impl->upper().stats(), u_info);
    });
}

int hec_precond_destroy(hec_precond_t m) {
    return guarded([&] { delete m; });
}

int hec_spmv_create(int n_rows, int n_cols, const int* row_offsets, const int* cols, const double* vals,
                    hec_spmv_t* out) {
    return guarded([&] {
        need(out, "hec_spmv_create");
        auto h = std::make_unique<hec_spmv>();
        h->impl = std::make_unique<hec::dev::DeviceSpmv>(n_rows, n_cols, row_offsets, cols, vals);
        *out = h.release();
    });
}

int hec_spmv_create_hec(int n_rows, int n_cols, int ell_width, const int* ell_cols, const double* ell_vals,
                        const int* csr_row_offsets, const int* csr_cols, const double* csr_vals, hec_spmv_t* out) {
    return guarded([&] {
        need(out, "hec_spmv_create_hec");
        if (n_rows > 0) need(csr_row_offsets, "hec_spmv_create_hec");
        auto h = std::make_unique<hec_spmv>();
        h->impl = std::make_unique<hec::dev::DeviceSpmv>(n_rows, n_cols, ell_width, ell_cols, ell_vals,
                                                         csr_row_offsets, csr_cols, csr_vals);
        *out = h.release();
    });
}

int hec_spmv_residual(hec_spmv_t a, const double* b_dev, const double* x_dev, double* y_dev, void* stream) {
    return guarded([&] {
        need(a, "hec_spmv_residual");
        a->impl->residual(b_dev, x_dev, y_dev, static_cast<cudaStream_t>(stream));
    });
}

int hec_spmv_run(hec_spmv_t a, const double* x_dev, double* y_dev, void* stream) {
    return guarded([&] {
        need(a, "hec_spmv_run");
        a->impl->run(x_dev, y_dev, static_cast<cudaStream_t>(stream));
    });
}

int hec_spmv_run_host(hec_spmv_t a, const double* x, double* y) {
    return guarded([&] {
        need(a, "hec_spmv_run_host");
        a->impl->run_host(x, y);
    });
}

int hec_spmv_destroy(hec_spmv_t a) {
    return guarded([&] { delete a; });
}

static void fill_report(const hec::dev::GmresOutcome& o, hec_gmres_report* report, double* inner, int cap) {
    if (report) {
        report->converged = o.converged ? 1 : 0;
        report->iterations = o.iterations;
        report->final_relative_residual = o.final_relative_residual;
        report->solve_seconds = o.solve_seconds;
        report->n_inner = static_cast<int>(o.inner_residuals.size());
    }
    if (inner)
        for (int k = 0; k < std::min<int>(cap, static_cast<int>(o.inner_residuals.size())); ++k)
            inner[k] = o.inner_residuals[k];
}

int hec_gmres_solve(hec_spmv_t a, hec_precond_t m, const double* b, const hec_gmres_config* cfg, double* x,
                    hec_gmres_report* report, double* inner_residuals, int inner_capacity) {
    return guarded([&] {
        need(a, "hec_gmres_solve");
        need(cfg, "hec_gmres_solve");
        hec::dev::GmresParams gp{cfg->restart, cfg->max_iters, cfg->rel_tol, cfg->abs_tol};
        const auto o = hec::dev::gmres_device(*a->impl, m ? m->impl.get() : nullptr, b, gp, x);
        fill_report(o, report, inner_residuals, inner_capacity);
    });
}

// ---- host setup ----
int hec_csr_create(int n_rows, int n_cols, const int* row_offsets, const int* cols, const double* vals,
                   hec_csr_t* out) {
    return guarded([&] {
        need(out, "hec_csr_create");
        if (n_rows < 0 || n_cols < 0) throw std::invalid_argument("hec_csr_create: negative dimension");
        auto h = std::make_unique<hec_csr>();
        h->m.n_rows = n_rows;
        h->m.n_cols = n_cols;
        h->m.row_offsets.assign(row_offsets, row_offsets + n_rows + 1);
        const int nnz = h->m.row_offsets[n_rows];
        h->m.col_indices.assign(cols, cols + nnz);
        h->m.values.assign(vals, vals + nnz);
        *out = h.release();
    });
}

int hec_csr_from_triples(int n_rows, int n_cols, long long count, const int* rows, const int* cols,
                         const double* vals, hec_csr_t* out) {
    return guarded([&] {
        need(out, "hec_csr_from_triples");
        std::vector<hec::Triplet> t(static_cast<std::size_t>(count));
        for (long long k = 0; k < count; ++k) t[k] = {rows[k], cols[k], vals[k]};
        auto h = std::make_unique<hec_csr>();
        h->m = hec::csr_from_triples(n_rows, n_cols, std::move(t));
        *out = h.release();
    });
}

int hec_csr_view(hec_csr_t a, int* n_rows, int* n_cols, long long* nnz, const int** row_offsets,
                 const int** cols, const double** vals) {
    return guarded([&] {
        need(a, "hec_csr_view");
        if (n_rows) *n_rows = a->m.n_rows;
        if (n_cols) *n_cols = a->m.n_cols;
        if (nnz) *nnz = static_cast<long long>(a->m.col_indices.size());
        if (row_offsets) *row_offsets = a->m.row_offsets.data();
        if (cols) *cols = a->m.col_indices.data();
        if (vals) *vals = a->m.values.data();
    });
}

int hec_csr_destroy(hec_csr_t a) {
    return guarded([&] { delete a; });
}

int hec_csr_spmv_host(hec_csr_t a, const double* x, double* y, int workers) {
    return guarded([&] {
        need(a, "hec_csr_spmv_host");
        std::vector<double> xv(x, x + a->m.n_cols);
        const std::vector<double> yv = hec::spmv_csr(a->m, xv, workers);
        std::copy(yv.begin(), yv.end(), y);
    });
}

int hec_hec_from_csr(hec_csr_t a, int triangular, int width_mode, int width, hec_hec_t* out) {
    return guarded([&] {
        need(a, "hec_hec_from_csr");
        need(out, "hec_hec_from_csr");
        auto h = std::make_unique<hec_hec>();
        h->m = hec::hec_from_csr(a->m, triangular != 0, policy_of(width_mode, width));
        *out = h.release();
    });
}

int hec_hec_view_get(hec_hec_t h, hec_hec_view* v) {
    return guarded([&] {
        need(h, "hec_hec_view_get");
        need(v, "hec_hec_view_get");
        const hec::HecMatrix& m = h->m;
        v->n_rows = m.n_rows;
        v->n_cols = m.n_cols;
        v->ell_width = m.ell.width;
        v->ell_cols = m.ell.col_indices.data();
        v->ell_vals = m.ell.values.data();
        v->csr_row_offsets = m.csr.row_offsets.data();
        v->csr_cols = m.csr.col_indices.data();
        v->csr_vals = m.csr.values.data();
        v->csr_nnz = static_cast<long long>(m.csr.col_indices.size());
    });
}

int hec_hec_spmv_host(hec_hec_t h, const double* x, double* y, int workers) {
    return guarded([&] {
        need(h, "hec_hec_spmv_host");
        std::vector<double> xv(x, x + h->m.n_cols);
        const std::vector<double> yv = hec::spmv_hec(h->m, xv, workers);
        std::copy(yv.begin(), yv.end(), y);
    });
}

int hec_hec_destroy(hec_hec_t h) {
    return guarded([&] { delete h; });
}

#define HEC_WRAP_GEN(expr)                     \
    return guarded([&] {                       \
        need(out, "generator");                \
        auto h = std::make_unique<hec_csr>();  \
        h->m = (expr);                         \
        *out = h.release();                    \
    })

int hec_gen_poisson7(int nx, int ny, int nz, hec_csr_t* out) { HEC_WRAP_GEN(hec::gen_poisson7(nx, ny, nz)); }
int hec_gen_poisson27(int nx, int ny, int nz, hec_csr_t* out) { HEC_WRAP_GEN(hec::gen_poisson27(nx, ny, nz)); }
int hec_gen_reservoir7(int nx, int ny, int nz, double sigma, double kz_ratio, uint64_t seed, hec_csr_t* out) {
    HEC_WRAP_GEN(hec::gen_reservoir7(nx, ny, nz, sigma, kz_ratio, seed));
}
int hec_permute_symmetric(hec_csr_t a, const int* perm, hec_csr_t* out) {
    need(a, "hec_permute_symmetric");
    HEC_WRAP_GEN(hec::permute_symmetric(a->m, std::vector<int>(perm, perm + a->m.n_rows)));
}

int hec_csr_submatrix(hec_csr_t a, const int* rows, int count, hec_csr_t* out) {
    return guarded([&] {
        need(a, "hec_csr_submatrix");
        need(out, "hec_csr_submatrix");
        if (count < 0 || (count > 0 && !rows)) throw std::invalid_argument("hec_csr_submatrix: bad row set");
        std::vector<int> r(rows, rows + count);
        for (int k = 0; k < count; ++k) {
            if (r[k] < 0 || r[k] >= a->m.n_rows) throw std::out_of_range("hec_csr_submatrix: row out of range");
            if (k && r[k] <= r[k - 1]) throw std::invalid_argument("hec_csr_submatrix: rows must ascend");
        }
        auto h = std::make_unique<hec_csr>();
        h->m = hec::extract_block(a->m, r);
        *out = h.release();
    });
}

int hec_partition_create(hec_csr_t a, int parts, int overlap, hec_partition_t* out) {
    return guarded([&] {
        need(a, "hec_partition_create");
        need(out, "hec_partition_create");
        const hec::Partition p = hec::partition_graph(a->m, parts);
        const auto ext = hec::extend_overlap(a->m, p, overlap);
        auto h = std::make_unique<hec_partition>();
        h->n = p.n;
        h->parts = p.n_parts;
        h->part_of = p.part_of;
        h->ext_offsets.assign(1, 0);
        for (const auto& e : ext) {
            h->ext_rows.insert(h->ext_rows.end(), e.begin(), e.end());
            h->ext_offsets.push_back(static_cast<int>(h->ext_rows.size()));
        }
        *out = h.release();
    });
}

int hec_partition_view(hec_partition_t p, int* n, int* parts, const int** part_of, const int** ext_offsets,
                       const int** ext_rows) {
    return guarded([&] {
        need(p, "hec_partition_view");
        if (n) *n = p->n;
        if (parts) *parts = p->parts;
        if (part_of) *part_of = p->part_of.data();
        if (ext_offsets) *ext_offsets = p->ext_offsets.data();
        if (ext_rows) *ext_rows = p->ext_rows.data();
    });
}

int hec_partition_destroy(hec_partition_t p) {
    return guarded([&] { delete p; });
}

int hec_random_ordering(int n, uint64_t seed, int* perm) {
    return guarded([&] {
        const auto p = hec::random_ordering(n, seed);
        std::copy(p.begin(), p.end(), perm);
    });
}

int hec_rcm_ordering(hec_csr_t a, int* perm) {
    return guarded([&] {
        need(a, "hec_rcm_ordering");
        const auto p = hec::rcm_ordering(a->m);
        std::copy(p.begin(), p.end(), perm);
    });
}

static int wrap_ilu(hec_csr_t* l, hec_csr_t* u, const hec::IluFactors& f) {
    auto hl = std::make_unique<hec_csr>();
    auto hu = std::make_unique<hec_csr>();
    hl->m = f.l;
    hu->m = f.u;
    *l = hl.release();
    *u = hu.release();
    return HEC_OK;
}

int hec_ilu0(hec_csr_t a, hec_csr_t* l, hec_csr_t* u) {
    return guarded([&] {
        need(a, "hec_ilu0");
        wrap_ilu(l, u, hec::ilu0(a->m));
    });
}
int hec_ilu_k(hec_csr_t a, int k, hec_csr_t* l, hec_csr_t* u) {
    return guarded([&] {
        need(a, "hec_ilu_k");
        wrap_ilu(l, u, hec::ilu_k(a->m, k));
    });
}
int hec_ilut(hec_csr_t a, int p, double tol, hec_csr_t* l, hec_csr_t* u) {
    return guarded([&] {
        need(a, "hec_ilut");
        wrap_ilu(l, u, hec::ilut(a->m, p, tol));
    });
}

int hec_prepare(hec_csr_t t, int upper, int width_mode, int width, hec_prep_t* out) {
    return guarded([&] {
        need(t, "hec_prepare");
        need(out, "hec_prepare");
        auto h = std::make_unique<hec_prep>();
        const hec::WidthPolicy pol = policy_of(width_mode, width);
        h->p = std::make_shared<const hec::PreparedTriangular>(upper ? hec::prepare_upper(t->m, pol)
                                                                     : hec::prepare_lower(t->m, pol));
        *out = h.release();
    });
}

int hec_prep_view_get(hec_prep_t h, hec_prep_view* v) {
    return guarded([&] {
        need(h, "hec_prep_view_get");
        need(v, "hec_prep_view_get");
        const hec::PreparedTriangular& p = *h->p;
        v->kind = p.kind == hec::TriKind::upper ? 1 : 0;
        v->n = p.n;
        v->reversal_applied = p.reversal_applied ? 1 : 0;
        v->nlev = p.schedule.nlev;
        v->level_of = p.schedule.level_of.data();
        v->perm = p.schedule.perm.data();
        v->inv_perm = p.schedule.inv_perm.data();
        v->level_starts = p.schedule.level_starts.data();
        v->ell_width = p.hec.ell.width;
        v->ell_cols = p.hec.ell.col_indices.data();
        v->ell_vals = p.hec.ell.values.data();
        v->csr_row_offsets = p.hec.csr.row_offsets.data();
        v->csr_cols = p.hec.csr.col_indices.data();
        v->csr_vals = p.hec.csr.values.data();
        v->csr_nnz = static_cast<long long>(p.hec.csr.col_indices.size());
    });
}

int hec_prep_solve_host(hec_prep_t h, const double* b, double* x) {
    return guarded([&] {
        need(h, "hec_prep_solve_host");
        std::vector<double> bv(b, b + h->p->n);
        const std::vector<double> xv = hec::solve(*h->p, bv);
        std::copy(xv.begin(), xv.end(), x);
    });
}

int hec_prep_device(hec_prep_t h, hec_tri_t* t) {
    return guarded([&] {
        need(h, "hec_prep_device");
        *t = hec::device_handle(*h->p);
        if (!*t) throw std::logic_error("hec_prep_device: device mirror belongs to another object");
    });
}

int hec_serial_solve(hec_csr_t t, int upper, const double* b, double* x) {
    return guarded([&] {
        need(t, "hec_serial_solve");
        std::vector<double> bv(b, b + t->m.n_rows);
        const std::vector<double> xv =
            upper ? hec::serial_backward_solve(t->m, bv) : hec::serial_forward_solve(t->m, bv);
        std::copy(xv.begin(), xv.end(), x);
    });
}

int hec_prep_destroy(hec_prep_t p) {
    return guarded([&] { delete p; });
}

int hec_bp_build(hec_csr_t a, int kind, int blocks, int overlap, int ilut_p, double ilut_tol, int width_mode,
                 int width, int fill_level, hec_bp_t* out) {
    return guarded([&] {
        need(a, "hec_bp_build");
        need(out, "hec_bp_build");
        if (kind < 0 || kind > 3) throw std::invalid_argument("hec_bp_build: unknown kind");
        auto h = std::make_unique<hec_bp>();
        h->m = hec::build_preconditioner(a->m, static_cast<hec::PrecondKind>(kind), blocks, overlap, ilut_p,
                                         ilut_tol, policy_of(width_mode, width), fill_level);
        // borrowed prepared views that alias the preconditioner's members
        std::shared_ptr<const hec::BlockPreconditioner> none;
        h->l.p = std::shared_ptr<const hec::PreparedTriangular>(none, &h->m.prepared_l);
        h->u.p = std::shared_ptr<const hec::PreparedTriangular>(none, &h->m.prepared_u);
        *out = h.release();
    });
}

int hec_bp_dims(hec_bp_t m, int* n, int* n_parts, int* n_ext) {
    return guarded([&] {
        need(m, "hec_bp_dims");
        if (n) *n = m->m.n;
        if (n_parts) *n_parts = m->m.partition.n_parts;
        if (n_ext) *n_ext = m->m.offsets.empty() ? 0 : m->m.offsets.back();
    });
}

int hec_bp_maps(hec_bp_t h, int* part_of, int* offsets, int* ext_rows, char* owned) {
    return guarded([&] {
        need(h, "hec_bp_maps");
        const hec::BlockPreconditioner& m = h->m;
        if (part_of) std::copy(m.partition.part_of.begin(), m.partition.part_of.end(), part_of);
        if (offsets) std::copy(m.offsets.begin(), m.offsets.end(), offsets);
        for (int p = 0; p < m.partition.n_parts; ++p) {
            if (ext_rows) std::copy(m.extended_parts[p].begin(), m.extended_parts[p].end(), ext_rows + m.offsets[p]);
            if (owned) std::copy(m.restriction[p].begin(), m.restriction[p].end(), owned + m.offsets[p]);
        }
    });
}

int hec_bp_prepared(hec_bp_t m, hec_prep_t* l, hec_prep_t* u) {
    return guarded([&] {
        need(m, "hec_bp_prepared");
        if (l) *l = &m->l;
        if (u) *u = &m->u;
    });
}

int hec_bp_apply_host(hec_bp_t m, const double* r, double* x) {
    return guarded([&] {
        need(m, "hec_bp_apply_host");
        std::vector<double> rv(r, r + m->m.n);
        const std::vector<double> xv = hec::apply(m->m, rv);
        std::copy(xv.begin(), xv.end(), x);
    });
}

int hec_bp_device(hec_bp_t m, hec_precond_t* d) {
    return guarded([&] {
        need(m, "hec_bp_device");
        *d = hec::device_handle(m->m);
        if (!*d) throw std::logic_error("hec_bp_device: device mirror belongs to another object");
    });
}

int hec_bp_destroy(hec_bp_t m) {
    return guarded([&] { delete m; });
}

int hec_gmres_host(hec_csr_t a, const double* b, hec_bp_t m, const hec_gmres_config* cfg, double* x,
                   hec_gmres_report* report, double* inner_residuals, int inner_capacity) {
    return guarded([&] {
        need(a, "hec_gmres_host");
        need(cfg, "hec_gmres_host");
        hec::SolverConfig c{cfg->restart, cfg->max_iters, cfg->rel_tol, cfg->abs_tol};
        std::vector<double> bv(b, b + a->m.n_rows);
        const hec::SolveResult res = hec::gmres(a->m, bv, m ? &m->m : nullptr, c);
        std::copy(res.x.begin(), res.x.end(), x);
        hec::dev::GmresOutcome o;
        o.converged = res.report.converged;
        o.iterations = res.report.iterations;
        o.final_relative_residual = res.report.final_relative_residual;
        o.solve_seconds = res.report.solve_seconds;
        o.inner_residuals = res.report.inner_residuals;
        fill_report(o, report, inner_residuals, inner_capacity);
    });
}

// ---- multi-GPU RAS ----
int hec_ras_plan_create(hec_csr_t a, int world, int rank, int overlap, hec_ras_plan_t* out) {
    return guarded([&] {
        need(a, "hec_ras_plan_create");
        need(out, "hec_ras_plan_create");
        auto h = std::make_unique<hec_ras_plan>();
        h->plan = hec::ras::make_plan(a->m, world, rank, overlap);
        *out = h.release();
    });
}

int hec_ras_plan_view_get(hec_ras_plan_t p, hec_ras_plan_view* v) {
    return guarded([&] {
        need(p, "hec_ras_plan_view_get");
        need(v, "hec_ras_plan_view_get");
        const hec::ras::Plan& P = p->plan;
        v->n = P.n;
        v->rank = P.rank;
        v->world = P.world;
        v->overlap = P.overlap;
        v->n_own = P.n_own();
        v->n_halo = static_cast<int>(P.halo.size());
        v->n_ext = static_cast<int>(P.ext.size());
        v->n_send = static_cast<int>(P.send_idx.size());
        v->own = P.own.data();
        v->halo = P.halo.data();
        v->ext = P.ext.data();
        v->send_offsets = P.send_offsets.data();
        v->send_idx = P.send_idx.data();
        v->recv_offsets = P.recv_offsets.data();
        v->gather = P.gather.data();
        v->out_index = P.out_index.data();
        v->part_of = P.part_of.data();
    });
}

int hec_ras_plan_destroy(hec_ras_plan_t p) {
    return guarded([&] { delete p; });
}

int hec_nccl_unique_id(unsigned char id[128]) {
    return guarded([&] {
        need(id, "hec_nccl_unique_id");
        hec::dev::nccl_unique_id(id);
    });
}

int hec_nccl_version(void) { return hec::dev::nccl_version(); }

int hec_ras_create(hec_csr_t a, int overlap, int local_kind, int ilut_p, double ilut_tol, int fill_level,
                   const hec_comm_spec* comm, hec_ras_t* out) {
    return guarded([&] {
        need(a, "hec_ras_create");
        need(out, "hec_ras_create");
        hec::dev::require_device();
        const int kind = comm ? comm->kind : HEC_COMM_NONE;
        const int world = kind == HEC_COMM_NONE ? 1 : comm->world;
        const int rank = kind == HEC_COMM_NONE ? 0 : comm->rank;
        auto h = std::make_unique<hec_ras>();
        h->p.plan = hec::ras::make_plan(a->m, world, rank, overlap);
        const hec::ras::Plan& P = h->p.plan;
        // the rank's block: the reference's per-part factorisation (precond.cpp:97-110)
        const hec::CsrMatrix blk = hec::extract_block(a->m, P.ext);
        hec::IluFactors f;
        try {
            f = local_kind == 1   ? hec::ilut(blk, ilut_p, ilut_tol)
                : local_kind == 3 ? hec::ilu_k(blk, fill_level)
                                  : hec::ilu0(blk);
        } catch (const hec::ZeroPivotError& e) {
            throw hec::ZeroPivotError(e.row(), rank);  // re-tagged with the block (precond.cpp:107-109)
        }
        const hec::PreparedTriangular pl = hec::prepare_lower(f.l), pu = hec::prepare_upper(f.u);
        h->M = std::make_unique<hec::dev::DevicePrecond>(P.n_loc(), P.n_own(), static_cast<int>(P.ext.size()),
                                                         P.gather.data(), P.out_index.data(), hec::source_of(pl),
                                                         hec::source_of(pu), hec::tri_options(nullptr));
        h->A = std::make_unique<hec::dev::DeviceSpmv>(P.a_local.n_rows, P.a_local.n_cols,
                                                      P.a_local.row_offsets.data(), P.a_local.col_indices.data(),
                                                      P.a_local.values.data());
        h->send_idx.upload(P.send_idx);
        if (kind == HEC_COMM_NCCL) {
            need(comm->nccl_id, "hec_ras_create (nccl_id)");
            h->comm = std::make_unique<hec::dev::NcclComm>(comm->nccl_id, rank, world);
        } else if (kind == HEC_COMM_CALLBACKS) {
            if (!comm->callbacks.allreduce_sum || !comm->callbacks.exchange)
                throw std::invalid_argument("hec_ras_create: missing callbacks");
            hec::dev::CommCallbacks cb;
            cb.ctx = comm->callbacks.ctx;
            cb.allreduce_sum = comm->callbacks.allreduce_sum;
            cb.exchange = comm->callbacks.exchange;
            h->comm = std::make_unique<hec::dev::CallbackComm>(cb, rank, world);
        } else if (kind == HEC_COMM_NONE) {
            h->comm = std::make_unique<hec::dev::NullComm>();
        } else {
            throw std::invalid_argument("hec_ras_create: unknown comm kind");
        }
        HEC_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        *out = h.release();
    });
}

int hec_ras_get_plan(hec_ras_t r, hec_ras_plan_t* plan) {
    return guarded([&] {
        need(r, "hec_ras_get_plan");
        need(plan, "hec_ras_get_plan");
        *plan = &r->p;
    });
}

namespace {
hec::dev::DistSystem ras_system(hec_ras_t r) {
    const hec::ras::Plan& P = r->p.plan;
    hec::dev::DistSystem S;
    S.n_own = P.n_own();
    S.n_loc = P.n_loc();
    S.A = r->A.get();
    S.M = r->M.get();
    S.send_idx = r->send_idx.p;
    S.n_send = static_cast<int>(P.send_idx.size());
    S.send_off = P.send_offsets;
    S.recv_off = P.recv_offsets;
    S.comm = r->comm.get();
    return S;
}
}  // namespace

int hec_ras_apply(hec_ras_t r, const double* r_own_dev, double* z_own_dev, void* stream) {
    return guarded([&] {
        need(r, "hec_ras_apply");
        const hec::ras::Plan& P = r->p.plan;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (r->vloc.count < static_cast<std::size_t>(std::max(P.n_loc(), 1))) r->vloc.alloc(std::max(P.n_loc(), 1));
        if (r->sendbuf.count < std::max<std::size_t>(P.send_idx.size(), 1)) r->sendbuf.alloc(std::max<std::size_t>(P.send_idx.size(), 1));
        HEC_CUDA(cudaMemcpyAsync(r->vloc.p, r_own_dev, sizeof(double) * P.n_own(), cudaMemcpyDeviceToDevice, st));
        hec::dev::halo_exchange(ras_system(r), r->vloc.p, r->sendbuf.p, st);
        r->M->apply(r->vloc.p, z_own_dev, st);
    });
}

int hec_ras_apply_host(hec_ras_t r, const double* r_own, double* z_own) {
    return guarded([&] {
        need(r, "hec_ras_apply_host");
        const int n = r->p.plan.n_own();
        if (r->h_r.count < static_cast<std::size_t>(std::max(n, 1))) {
            r->h_r.alloc(std::max(n, 1));
            r->h_z.alloc(std::max(n, 1));
        }
        HEC_CUDA(cudaMemcpyAsync(r->h_r.p, r_own, sizeof(double) * n, cudaMemcpyHostToDevice, r->stream));
        if (hec_ras_apply(r, r->h_r.p, r->h_z.p, r->stream) != HEC_OK) throw std::runtime_error(t_msg);
        HEC_CUDA(cudaMemcpyAsync(z_own, r->h_z.p, sizeof(double) * n, cudaMemcpyDeviceToHost, r->stream));
        HEC_CUDA(cudaStreamSynchronize(r->stream));
    });
}

int hec_ras_gmres_device(hec_ras_t r, const double* b_own_dev, const hec_gmres_config* cfg, double* x_own_dev,
                         hec_gmres_report* report, double* inner_residuals, int inner_capacity, void* stream) {
    return guarded([&] {
        need(r, "hec_ras_gmres_device");
        need(cfg, "hec_ras_gmres_device");
        hec::dev::GmresParams gp{cfg->restart, cfg->max_iters, cfg->rel_tol, cfg->abs_tol};
        hec::dev::DistSystem S = ras_system(r);
        const long long a0 = r->comm->allreduces, e0 = r->comm->exchanges;
        const auto o = hec::dev::gmres_dist(S, b_own_dev, x_own_dev, gp, static_cast<cudaStream_t>(stream));
        r->allreduces = r->comm->allreduces - a0;
        r->exchanges = r->comm->exchanges - e0;
        r->launches = o.launches;
        fill_report(o, report, inner_residuals, inner_capacity);
    });
}

int hec_ras_gmres(hec_ras_t r, const double* b_own, const hec_gmres_config* cfg, double* x_own,
                  hec_gmres_report* report, double* inner_residuals, int inner_capacity) {
    return guarded([&] {
        need(r, "hec_ras_gmres");
        const int n = r->p.plan.n_own();
        hec::dev::DevBuf<double> b(std::max(n, 1)), x(std::max(n, 1));
        HEC_CUDA(cudaMemcpyAsync(b.p, b_own, sizeof(double) * n, cudaMemcpyHostToDevice, r->stream));
        const int rc = hec_ras_gmres_device(r, b.p, cfg, x.p, report, inner_residuals, inner_capacity, r->stream);
        if (rc != HEC_OK) throw std::runtime_error(t_msg);
        HEC_CUDA(cudaMemcpyAsync(x_own, x.p, sizeof(double) * n, cudaMemcpyDeviceToHost, r->stream));
        HEC_CUDA(cudaStreamSynchronize(r->stream));
    });
}

int hec_ras_stats(hec_ras_t r, long long* allreduces, long long* exchanges, long long* launches) {
    return guarded([&] {
        need(r, "hec_ras_stats");
        if (allreduces) *allreduces = r->allreduces;
        if (exchanges) *exchanges = r->exchanges;
        if (launches) *launches = r->launches;
    });
}

int hec_ras_destroy(hec_ras_t r) {
    return guarded([&] { delete r; });
}

}  // extern "C"
