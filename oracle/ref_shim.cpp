// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY. A C-ABI over the UNMODIFIED
// reference library (/root/reference/proj/src), compiled together with it into
// oracle/_ref/libhecref.so by oracle/Makefile with -Dhec=hecref so it can share
// a process with the product. Used by tests/ (CPU parity of the host setup,
// golden-vector generation) and by bench.py --impl reference / cpu_baseline.
// No reference source is copied: the reference .cpp files are compiled from
// where they lie, and its test helpers are #included from there.

#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "hecsolve/csr.hpp"
#include "hecsolve/errors.hpp"
#include "hecsolve/gmres.hpp"
#include "hecsolve/ilu.hpp"
#include "hecsolve/level_schedule.hpp"
#include "hecsolve/poisson.hpp"
#include "hecsolve/precond.hpp"
#include "hecsolve/triangular.hpp"
#include "test_helpers.hpp"

namespace {

// A bag of named arrays plus the live reference objects they came from.
struct Bag {
    std::map<std::string, std::vector<int>> ints;
    std::map<std::string, std::vector<double>> dbls;
    std::map<std::string, std::vector<char>> chars;
    std::shared_ptr<hecref::PreparedTriangular> prep;
    std::shared_ptr<hecref::BlockPreconditioner> bp;
    std::shared_ptr<hecref::CsrMatrix> csr;
};

thread_local std::string g_err;
thread_local int g_row = -1, g_block = -1;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const hecref::ZeroPivotError& e) {
        g_err = e.what();
        g_row = e.row();
        g_block = e.block();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

hecref::CsrMatrix csr_in(int nr, int nc, const int* rp, const int* ci, const double* v) {
    hecref::CsrMatrix a;
    a.n_rows = nr;
    a.n_cols = nc;
    a.row_offsets.assign(rp, rp + nr + 1);
    a.col_indices.assign(ci, ci + rp[nr]);
    a.values.assign(v, v + rp[nr]);
    return a;
}

void put_csr(Bag& b, const std::string& p, const hecref::CsrMatrix& m) {
    b.ints[p + "dims"] = {m.n_rows, m.n_cols};
    b.ints[p + "rp"] = m.row_offsets;
    b.ints[p + "ci"] = m.col_indices;
    b.dbls[p + "v"] = m.values;
}

void put_prep(Bag& b, const std::string& p, const hecref::PreparedTriangular& t) {
    b.ints[p + "meta"] = {t.kind == hecref::TriKind::upper ? 1 : 0, t.n, t.reversal_applied ? 1 : 0,
                          t.schedule.nlev, t.hec.ell.width};
    b.ints[p + "level_of"] = t.schedule.level_of;
    b.ints[p + "perm"] = t.schedule.perm;
    b.ints[p + "inv_perm"] = t.schedule.inv_perm;
    b.ints[p + "level_starts"] = t.schedule.level_starts;
    b.ints[p + "ell_cols"] = t.hec.ell.col_indices;
    b.dbls[p + "ell_vals"] = t.hec.ell.values;
    b.ints[p + "csr_rp"] = t.hec.csr.row_offsets;
    b.ints[p + "csr_ci"] = t.hec.csr.col_indices;
    b.dbls[p + "csr_v"] = t.hec.csr.values;
}

hecref::WidthPolicy pol(int mode, int w) {
    return mode == 1 ? hecref::WidthPolicy::fixed(w) : hecref::WidthPolicy::automatic();
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err.c_str(); }
__attribute__((visibility("default"))) int ref_last_error_row() { return g_row; }
__attribute__((visibility("default"))) int ref_last_error_block() { return g_block; }

__attribute__((visibility("default"))) void ref_free(void* h) { delete static_cast<Bag*>(h); }

// name lookups: return element count (or -1 when absent) and the data pointer
__attribute__((visibility("default"))) long long ref_get_int(void* h, const char* name, const int** out) {
    auto& m = static_cast<Bag*>(h)->ints;
    auto it = m.find(name);
    if (it == m.end()) return -1;
    *out = it->second.data();
    return static_cast<long long>(it->second.size());
}
__attribute__((visibility("default"))) long long ref_get_dbl(void* h, const char* name, const double** out) {
    auto& m = static_cast<Bag*>(h)->dbls;
    auto it = m.find(name);
    if (it == m.end()) return -1;
    *out = it->second.data();
    return static_cast<long long>(it->second.size());
}
__attribute__((visibility("default"))) long long ref_get_chr(void* h, const char* name, const char** out) {
    auto& m = static_cast<Bag*>(h)->chars;
    auto it = m.find(name);
    if (it == m.end()) return -1;
    *out = it->second.data();
    return static_cast<long long>(it->second.size());
}

// ---- generators (reference poisson.cpp and tests/test_helpers.hpp) ----
__attribute__((visibility("default"))) int ref_poisson7(int nx, int ny, int nz, void** out) {
    return guard([&] {
        auto b = std::make_unique<Bag>();
        b->csr = std::make_shared<hecref::CsrMatrix>(hecref::gen_poisson7(nx, ny, nz));
        put_csr(*b, "", *b->csr);
        *out = b.release();
    });
}

__attribute__((visibility("default"))) void* ref_rng_new(unsigned seed) { return new std::mt19937(seed); }
__attribute__((visibility("default"))) void ref_rng_free(void* r) { delete static_cast<std::mt19937*>(r); }
__attribute__((visibility("default"))) int ref_rng_int(void* r, int lo, int hi) {
    return std::uniform_int_distribution<int>(lo, hi)(*static_cast<std::mt19937*>(r));
}
__attribute__((visibility("default"))) double ref_rng_real(void* r, double lo, double hi) {
    return std::uniform_real_distribution<double>(lo, hi)(*static_cast<std::mt19937*>(r));
}
__attribute__((visibility("default"))) void ref_random_vector(void* r, int n, double* out) {
    const auto v = hecref::test::random_vector(n, *static_cast<std::mt19937*>(r));
    std::memcpy(out, v.data(), sizeof(double) * n);
}
// kind: 0 lower, 1 upper, 2 diagonally dominant
__attribute__((visibility("default"))) int ref_random_matrix(void* r, int kind, int n, double density, void** out) {
    return guard([&] {
        auto& rng = *static_cast<std::mt19937*>(r);
        auto b = std::make_unique<Bag>();
        b->csr = std::make_shared<hecref::CsrMatrix>(kind == 0   ? hecref::test::random_lower(n, density, rng)
                                                     : kind == 1 ? hecref::test::random_upper(n, density, rng)
                                                                 : hecref::test::random_diag_dominant(n, density, rng));
        put_csr(*b, "", *b->csr);
        *out = b.release();
    });
}

// ---- the path ----
__attribute__((visibility("default"))) int ref_prepare(int n, const int* rp, const int* ci, const double* v,
                                                       int upper, int wmode, int w, void** out) {
    return guard([&] {
        const hecref::CsrMatrix a = csr_in(n, n, rp, ci, v);
        auto b = std::make_unique<Bag>();
        b->prep = std::make_shared<hecref::PreparedTriangular>(upper ? hecref::prepare_upper(a, pol(wmode, w))
                                                                     : hecref::prepare_lower(a, pol(wmode, w)));
        put_prep(*b, "", *b->prep);
        *out = b.release();
    });
}

// Rebuild a reference PreparedTriangular from arrays (e.g. the product's own
// setup output, already proven identical) without re-running setup.
__attribute__((visibility("default"))) int ref_prepared_from_arrays(
    int kind, int n, int reversed, int nlev, const int* level_of, const int* perm, const int* inv_perm,
    const int* level_starts, int w, const int* ell_cols, const double* ell_vals, const int* csr_rp,
    const int* csr_ci, const double* csr_v, void** out) {
    return guard([&] {
        auto t = std::make_shared<hecref::PreparedTriangular>();
        t->kind = kind ? hecref::TriKind::upper : hecref::TriKind::lower;
        t->n = n;
        t->reversal_applied = reversed != 0;
        t->schedule.n = n;
        t->schedule.nlev = nlev;
        t->schedule.level_of.assign(level_of, level_of + n);
        t->schedule.perm.assign(perm, perm + n);
        t->schedule.inv_perm.assign(inv_perm, inv_perm + n);
        t->schedule.level_starts.assign(level_starts, level_starts + nlev + 1);
        t->hec.n_rows = t->hec.n_cols = n;
        t->hec.ell.n_rows = n;
        t->hec.ell.width = w;
        t->hec.ell.col_indices.assign(ell_cols, ell_cols + static_cast<std::size_t>(w) * n);
        t->hec.ell.values.assign(ell_vals, ell_vals + static_cast<std::size_t>(w) * n);
        t->hec.csr = csr_in(n, n, csr_rp, csr_ci, csr_v);
        auto b = std::make_unique<Bag>();
        b->prep = t;
        *out = b.release();
    });
}

__attribute__((visibility("default"))) int ref_solve(void* prep, const double* bvec, double* x, int workers) {
    return guard([&] {
        const Bag* b = static_cast<Bag*>(prep);
        const std::vector<double> rhs(bvec, bvec + b->prep->n);
        const std::vector<double> y = hecref::solve(*b->prep, rhs, workers);
        std::memcpy(x, y.data(), sizeof(double) * y.size());
    });
}

__attribute__((visibility("default"))) int ref_serial_solve(int n, const int* rp, const int* ci, const double* v,
                                                            int upper, const double* bvec, double* x) {
    return guard([&] {
        const hecref::CsrMatrix a = csr_in(n, n, rp, ci, v);
        const std::vector<double> rhs(bvec, bvec + n);
        const std::vector<double> y =
            upper ? hecref::serial_backward_solve(a, rhs) : hecref::serial_forward_solve(a, rhs);
        std::memcpy(x, y.data(), sizeof(double) * y.size());
    });
}

__attribute__((visibility("default"))) int ref_spmv(int nr, int nc, const int* rp, const int* ci, const double* v,
                                                    const double* x, double* y, int workers) {
    return guard([&] {
        const hecref::CsrMatrix a = csr_in(nr, nc, rp, ci, v);
        const std::vector<double> xv(x, x + nc);
        const std::vector<double> yv = hecref::spmv_csr(a, xv, workers);
        std::memcpy(y, yv.data(), sizeof(double) * yv.size());
    });
}

// kind: 0 ilu0, 1 ilu_k(k), 2 ilut(p, tol)
__attribute__((visibility("default"))) int ref_ilu(int n, const int* rp, const int* ci, const double* v, int kind,
                                                   int k_or_p, double tol, void** out) {
    return guard([&] {
        const hecref::CsrMatrix a = csr_in(n, n, rp, ci, v);
        const hecref::IluFactors f = kind == 0   ? hecref::ilu0(a)
                                     : kind == 1 ? hecref::ilu_k(a, k_or_p)
                                                 : hecref::ilut(a, k_or_p, tol);
        auto b = std::make_unique<Bag>();
        put_csr(*b, "l_", f.l);
        put_csr(*b, "u_", f.u);
        *out = b.release();
    });
}

// kind: 0 bilu0, 1 bilut, 2 ras
__attribute__((visibility("default"))) int ref_precond(int n, const int* rp, const int* ci, const double* v, int kind,
                                                       int blocks, int overlap, int p, double tol, int wmode, int w,
                                                       void** out) {
    return guard([&] {
        const hecref::CsrMatrix a = csr_in(n, n, rp, ci, v);
        auto b = std::make_unique<Bag>();
        b->bp = std::make_shared<hecref::BlockPreconditioner>(hecref::build_preconditioner(
            a, static_cast<hecref::PrecondKind>(kind), blocks, overlap, p, tol, pol(wmode, w)));
        const auto& m = *b->bp;
        b->ints["part_of"] = m.partition.part_of;
        b->ints["offsets"] = m.offsets;
        std::vector<int> ext;
        std::vector<char> own;
        for (int q = 0; q < m.partition.n_parts; ++q) {
            ext.insert(ext.end(), m.extended_parts[q].begin(), m.extended_parts[q].end());
            own.insert(own.end(), m.restriction[q].begin(), m.restriction[q].end());
        }
        b->ints["ext_rows"] = ext;
        b->chars["owned"] = own;
        put_prep(*b, "l_", m.prepared_l);
        put_prep(*b, "u_", m.prepared_u);
        *out = b.release();
    });
}

// A single-block BlockPreconditioner holding the given factors (the hand
// assembly SURVEY.md 8(b) describes for ILU(k), which PrecondKind lacks):
// apply() reads only n, partition.n_parts, extended_parts, offsets,
// restriction and prepared_l/u (precond.cpp:119-145).
__attribute__((visibility("default"))) int ref_precond_single(int n, const int* lrp, const int* lci, const double* lv,
                                                              const int* urp, const int* uci, const double* uv,
                                                              void** out) {
    return guard([&] {
        auto b = std::make_unique<Bag>();
        auto m = std::make_shared<hecref::BlockPreconditioner>();
        m->kind = hecref::PrecondKind::bilu0;
        m->n = n;
        m->partition.n = n;
        m->partition.n_parts = 1;
        m->partition.part_of.assign(n, 0);
        std::vector<int> rows(n);
        for (int i = 0; i < n; ++i) rows[i] = i;
        m->partition.parts = {rows};
        m->extended_parts = {rows};
        m->restriction = {std::vector<char>(n, 1)};
        m->offsets = {0, n};
        const hecref::CsrMatrix l = csr_in(n, n, lrp, lci, lv), u = csr_in(n, n, urp, uci, uv);
        m->prepared_l = hecref::prepare_lower(l);
        m->prepared_u = hecref::prepare_upper(u);
        b->bp = m;
        *out = b.release();
    });
}

__attribute__((visibility("default"))) int ref_apply(void* bp, const double* r, double* x, int workers) {
    return guard([&] {
        const Bag* b = static_cast<Bag*>(bp);
        const std::vector<double> rv(r, r + b->bp->n);
        const std::vector<double> xv = hecref::apply(*b->bp, rv, workers);
        std::memcpy(x, xv.data(), sizeof(double) * xv.size());
    });
}

// report: [converged, iterations, final_rel_res, solve_seconds, n_inner]
__attribute__((visibility("default"))) int ref_gmres(int n, const int* rp, const int* ci, const double* v,
                                                     const double* bvec, void* bp, int restart, int max_iters,
                                                     double rel_tol, double abs_tol, int workers, double* x,
                                                     double* report) {
    return guard([&] {
        const hecref::CsrMatrix a = csr_in(n, n, rp, ci, v);
        const std::vector<double> rhs(bvec, bvec + n);
        hecref::SolverConfig cfg{restart, max_iters, rel_tol, abs_tol};
        const hecref::BlockPreconditioner* m = bp ? static_cast<Bag*>(bp)->bp.get() : nullptr;
        const hecref::SolveResult res = hecref::gmres(a, rhs, m, cfg, workers);
        std::memcpy(x, res.x.data(), sizeof(double) * n);
        report[0] = res.report.converged ? 1.0 : 0.0;
        report[1] = res.report.iterations;
        report[2] = res.report.final_relative_residual;
        report[3] = res.report.solve_seconds;
        report[4] = static_cast<double>(res.report.inner_residuals.size());
    });
}

}  // extern "C"
