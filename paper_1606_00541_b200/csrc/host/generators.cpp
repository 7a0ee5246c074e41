// Matrix generators and orderings for the benchmark configurations.
// gen_poisson7 matches reference proj/src/poisson.cpp:8-43 entry for entry
// (x-fastest numbering, ascending columns, diag 6, int32 overflow check).
// gen_poisson27 / gen_reservoir7 / orderings are new; their definitions are the
// ones fixed in SURVEY.md §8(d) (configs C2, C3, C5).

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#include "hecsolve/partition.hpp"
#include "hecsolve/poisson.hpp"

namespace hec {

namespace {

void check_grid(const char* who, int nx, int ny, int nz, long long nnz_bound) {
    if (nx < 1 || ny < 1 || nz < 1)
        throw std::invalid_argument(std::string(who) + ": grid dimensions must be >= 1");
    const long long n = static_cast<long long>(nx) * ny * nz;
    if (n > std::numeric_limits<int>::max() || nnz_bound > std::numeric_limits<int>::max())
        throw std::overflow_error(std::string(who) + ": index range overflow");
}

}  // namespace

CsrMatrix gen_poisson7(int nx, int ny, int nz) {
    const long long n = static_cast<long long>(nx) * ny * nz;
    const long long nnz = 7 * n - 2 * (static_cast<long long>(nx) * ny +
                                       static_cast<long long>(ny) * nz +
                                       static_cast<long long>(nx) * nz);
    check_grid("gen_poisson7", nx, ny, nz, nnz);
    CsrMatrix m;
    m.n_rows = m.n_cols = static_cast<int>(n);
    m.row_offsets.resize(static_cast<std::size_t>(n) + 1);
    m.col_indices.resize(static_cast<std::size_t>(nnz));
    m.values.resize(static_cast<std::size_t>(nnz));
    const long long plane = static_cast<long long>(nx) * ny;
    long long at = 0;
    int id = 0;
    m.row_offsets[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++id) {
                auto put = [&](long long c, double v) {
                    m.col_indices[at] = static_cast<int>(c);
                    m.values[at] = v;
                    ++at;
                };
                if (z > 0) put(id - plane, -1.0);
                if (y > 0) put(id - nx, -1.0);
                if (x > 0) put(id - 1, -1.0);
                put(id, 6.0);
                if (x + 1 < nx) put(id + 1, -1.0);
                if (y + 1 < ny) put(id + nx, -1.0);
                if (z + 1 < nz) put(id + plane, -1.0);
                m.row_offsets[id + 1] = static_cast<int>(at);
            }
    return m;
}

CsrMatrix gen_poisson27(int nx, int ny, int nz) {
    auto span = [](long long d) { return 3 * d - 2 * (d > 1 ? 1 : 0) - (d == 1 ? 2 : 0); };
    // stored entries per axis: sum over cells of (#existing neighbours incl. self)
    const long long nnz = span(nx) * span(ny) * span(nz);
    check_grid("gen_poisson27", nx, ny, nz, nnz);
    const long long n = static_cast<long long>(nx) * ny * nz;
    CsrMatrix m;
    m.n_rows = m.n_cols = static_cast<int>(n);
    m.row_offsets.resize(static_cast<std::size_t>(n) + 1);
    m.col_indices.resize(static_cast<std::size_t>(nnz));
    m.values.resize(static_cast<std::size_t>(nnz));
    long long at = 0;
    int id = 0;
    m.row_offsets[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++id) {
                for (int dz = -1; dz <= 1; ++dz) {
                    if (z + dz < 0 || z + dz >= nz) continue;
                    for (int dy = -1; dy <= 1; ++dy) {
                        if (y + dy < 0 || y + dy >= ny) continue;
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (x + dx < 0 || x + dx >= nx) continue;
                            const long long c = id + dx + static_cast<long long>(nx) * (dy + static_cast<long long>(ny) * dz);
                            m.col_indices[at] = static_cast<int>(c);
                            m.values[at] = (dx | dy | dz) == 0 ? 26.0 : -1.0;
                            ++at;
                        }
                    }
                }
                m.row_offsets[id + 1] = static_cast<int>(at);
            }
    if (at != nnz) throw std::logic_error("gen_poisson27: entry count mismatch");
    return m;
}

CsrMatrix gen_reservoir7(int nx, int ny, int nz, double sigma, double kz_ratio, std::uint64_t seed) {
    const long long n = static_cast<long long>(nx) * ny * nz;
    const long long nnz = 7 * n - 2 * (static_cast<long long>(nx) * ny +
                                       static_cast<long long>(ny) * nz +
                                       static_cast<long long>(nx) * nz);
    check_grid("gen_reservoir7", nx, ny, nz, nnz);
    std::vector<double> k(static_cast<std::size_t>(n));
    std::mt19937_64 rng(seed);
    for (auto& kc : k) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        kc = std::pow(10.0, sigma * (2.0 * u - 1.0));
    }
    auto harmonic = [](double a, double b) { return 2.0 * a * b / (a + b); };
    const long long plane = static_cast<long long>(nx) * ny;
    CsrMatrix m;
    m.n_rows = m.n_cols = static_cast<int>(n);
    m.row_offsets.resize(static_cast<std::size_t>(n) + 1);
    m.col_indices.resize(static_cast<std::size_t>(nnz));
    m.values.resize(static_cast<std::size_t>(nnz));
    long long at = 0;
    int id = 0;
    m.row_offsets[0] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x, ++id) {
                const double kh = k[id], kv = kz_ratio * k[id];
                // faces in column order: z-, y-, x-, x+, y+, z+
                const bool has[6] = {z > 0, y > 0, x > 0, x + 1 < nx, y + 1 < ny, z + 1 < nz};
                const long long nb[6] = {id - plane, id - nx, id - 1, id + 1, id + nx, id + plane};
                double t[6];
                for (int f = 0; f < 6; ++f) {
                    const bool vertical = (f == 0 || f == 5);
                    const double own = vertical ? kv : kh;
                    t[f] = has[f] ? harmonic(own, vertical ? kz_ratio * k[nb[f]] : k[nb[f]]) : own;
                }
                double d = 0.0;
                for (int f = 0; f < 6; ++f) d += t[f];
                auto put = [&](long long c, double v) {
                    m.col_indices[at] = static_cast<int>(c);
                    m.values[at] = v;
                    ++at;
                };
                for (int f = 0; f < 3; ++f)
                    if (has[f]) put(nb[f], -t[f]);
                put(id, d);
                for (int f = 3; f < 6; ++f)
                    if (has[f]) put(nb[f], -t[f]);
                m.row_offsets[id + 1] = static_cast<int>(at);
            }
    return m;
}

CsrMatrix permute_symmetric(const CsrMatrix& a, const std::vector<int>& perm) {
    if (a.n_rows != a.n_cols || static_cast<int>(perm.size()) != a.n_rows)
        throw std::invalid_argument("permute_symmetric: size mismatch");
    const int n = a.n_rows;
    std::vector<int> inv(n);
    for (int i = 0; i < n; ++i) inv[perm[i]] = i;
    CsrMatrix b;
    b.n_rows = b.n_cols = n;
    b.row_offsets.assign(static_cast<std::size_t>(n) + 1, 0);
    for (int r = 0; r < n; ++r)
        b.row_offsets[r + 1] = b.row_offsets[r] + (a.row_offsets[inv[r] + 1] - a.row_offsets[inv[r]]);
    b.col_indices.resize(a.col_indices.size());
    b.values.resize(a.values.size());
#pragma omp parallel for schedule(dynamic, 4096)
    for (int r = 0; r < n; ++r) {
        const int i = inv[r];
        const int lo = a.row_offsets[i], len = a.row_offsets[i + 1] - lo;
        std::vector<std::pair<int, double>> row(len);
        for (int t = 0; t < len; ++t) row[t] = {perm[a.col_indices[lo + t]], a.values[lo + t]};
        std::sort(row.begin(), row.end(),
                  [](const auto& x, const auto& y) { return x.first < y.first; });
        for (int t = 0; t < len; ++t) {
            b.col_indices[b.row_offsets[r] + t] = row[t].first;
            b.values[b.row_offsets[r] + t] = row[t].second;
        }
    }
    return b;
}

std::vector<int> random_ordering(int n, std::uint64_t seed) {
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::mt19937_64 rng(seed);
    std::shuffle(perm.begin(), perm.end(), rng);
    return perm;
}

std::vector<int> rcm_ordering(const CsrMatrix& a) {
    const auto adj = symmetrized_adjacency(a);
    const int n = a.n_rows;
    std::vector<int> order;
    order.reserve(n);
    std::vector<int> dist(n, -1);
    std::vector<char> placed(n, 0);
    auto degree = [&](int v) { return static_cast<int>(adj[v].size()); };

    // BFS over unplaced vertices; returns the eccentricity of root and the
    // minimum-degree (then lowest-index) vertex of the last level.
    std::vector<int> q;
    auto sweep = [&](int root, int& far) {
        q.assign(1, root);
        dist[root] = 0;
        for (std::size_t h = 0; h < q.size(); ++h)
            for (int u : adj[q[h]])
                if (!placed[u] && dist[u] < 0) {
                    dist[u] = dist[q[h]] + 1;
                    q.push_back(u);
                }
        const int ecc = dist[q.back()];
        far = -1;
        for (int v : q) {
            if (dist[v] == ecc &&
                (far < 0 || degree(v) < degree(far) || (degree(v) == degree(far) && v < far)))
                far = v;
            dist[v] = -1;
        }
        return ecc;
    };

    std::vector<int> nb;
    for (int s = 0; s < n; ++s) {
        if (placed[s]) continue;
        int root = s, far = -1;
        int ecc = sweep(root, far);
        while (far != root) {  // George-Liu pseudo-peripheral search
            int far2 = -1;
            const int e2 = sweep(far, far2);
            if (e2 <= ecc) break;
            root = far;
            ecc = e2;
            far = far2;
        }
        const std::size_t first = order.size();
        order.push_back(root);
        placed[root] = 1;
        for (std::size_t h = first; h < order.size(); ++h) {
            nb.clear();
            for (int u : adj[order[h]])
                if (!placed[u]) nb.push_back(u);
            std::sort(nb.begin(), nb.end(), [&](int x, int y) {
                return degree(x) != degree(y) ? degree(x) < degree(y) : x < y;
            });
            for (int u : nb) {
                placed[u] = 1;
                order.push_back(u);
            }
        }
    }
    std::reverse(order.begin(), order.end());
    std::vector<int> perm(n);
    for (int r = 0; r < n; ++r) perm[order[r]] = r;
    return perm;
}

}  // namespace hec
