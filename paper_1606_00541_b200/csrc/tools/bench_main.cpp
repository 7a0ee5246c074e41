// hecsolve_bench: the reference's benchmark command line (proj/tools/bench_main.cpp,
// which needs CLI11) over this library -- same options and defaults, argv parsed by hand.
//
//   hecsolve_bench --matrix poisson:NX,NY,NZ|mm:PATH [--precond bilu0|ras|bilut:P,TOL]
//                  [--blocks 16] [--overlap 0] [--workers 4] [--restart 20]
//                  [--tol 1e-6] [--max-iters 10000] [--out results.csv]

#include <cstdio>
#include <cstdlib>
#include <exception>
#include <map>
#include <string>

#include "hecsolve/bench.hpp"

namespace {

int usage(const char* why) {
    std::fprintf(stderr, "hecsolve_bench: %s\nusage: hecsolve_bench --matrix SOURCE [--precond P] [--blocks N] "
                         "[--overlap N] [--workers N] [--restart N] [--tol X] [--max-iters N] [--out PATH]\n",
                 why);
    return 2;
}

bool to_int(const std::string& s, int& v) {
    char* end = nullptr;
    const long x = std::strtol(s.c_str(), &end, 10);
    if (s.empty() || *end) return false;
    v = static_cast<int>(x);
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    std::map<std::string, std::string> opt = {{"--precond", "bilu0"}, {"--out", "results.csv"},
                                              {"--blocks", "16"},     {"--overlap", "0"},
                                              {"--workers", "4"},     {"--restart", "20"},
                                              {"--max-iters", "10000"}, {"--tol", "1e-6"}};
    std::string matrix;
    for (int k = 1; k < argc; ++k) {
        const std::string key = argv[k];
        if (key == "-h" || key == "--help") return usage("help"), 0;
        if (k + 1 >= argc) return usage(("missing value for " + key).c_str());
        if (key == "--matrix")
            matrix = argv[++k];
        else if (opt.count(key))
            opt[key] = argv[++k];
        else
            return usage(("unknown option " + key).c_str());
    }
    if (matrix.empty()) return usage("--matrix is required");
    int blocks, overlap, workers, restart, max_iters;
    if (!to_int(opt["--blocks"], blocks) || !to_int(opt["--overlap"], overlap) ||
        !to_int(opt["--workers"], workers) || !to_int(opt["--restart"], restart) ||
        !to_int(opt["--max-iters"], max_iters))
        return usage("integer option expected");
    char* end = nullptr;
    const double tol = std::strtod(opt["--tol"].c_str(), &end);
    if (*end) return usage("--tol expects a number");
    try {
        const hec::CsrMatrix a = hec::load_matrix_spec(matrix);
        const hec::PrecondSpec spec = hec::parse_precond_spec(opt["--precond"]);
        hec::SolverConfig cfg;
        cfg.restart = restart;
        cfg.max_iters = max_iters;
        cfg.rel_tol = tol;
        std::printf("matrix %s: n=%d nnz=%lld\n", matrix.c_str(), a.n_rows, static_cast<long long>(a.nnz()));
        const hec::BenchRow row = hec::run_benchmark(a, spec, blocks, overlap, workers, cfg);
        hec::write_bench_csv({row}, opt["--out"]);
        std::printf("%s\n%s\n", hec::bench_csv_header().c_str(), hec::bench_csv_row(row).c_str());
        if (!row.converged) std::printf("note: solver did not converge within the limits\n");
        std::printf("wrote %s\n", opt["--out"].c_str());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
