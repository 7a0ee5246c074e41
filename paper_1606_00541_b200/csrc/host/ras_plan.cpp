// RAS plan of one rank (see ras_plan.hpp).

#include "ras_plan.hpp"

#include <algorithm>
#include <stdexcept>

#include "hecsolve/partition.hpp"

namespace hec::ras {

namespace {

// Rows rank p needs but does not own: ext_p u cols(A[own_p, :]) \ own_p,
// ordered by (owner, row).
std::vector<int> halo_of(const CsrMatrix& a, const Partition& part, const std::vector<int>& ext, int p,
                         std::vector<char>& mark) {
    std::vector<int> need;
    auto add = [&](int r) {
        if (part.part_of[r] != p && !mark[r]) {
            mark[r] = 1;
            need.push_back(r);
        }
    };
    for (int r : ext) add(r);
    for (int r : part.parts[p])
        for (int k = a.row_offsets[r]; k < a.row_offsets[r + 1]; ++k) add(a.col_indices[k]);
    for (int r : need) mark[r] = 0;
    std::sort(need.begin(), need.end(), [&](int x, int y) {
        return part.part_of[x] != part.part_of[y] ? part.part_of[x] < part.part_of[y] : x < y;
    });
    return need;
}

}  // namespace

Plan make_plan(const CsrMatrix& a, int world, int rank, int overlap) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("ras plan: matrix must be square");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("ras plan: bad rank / world");
    if (overlap < 0) throw std::invalid_argument("ras plan: overlap must be >= 0");
    const int n = a.n_rows;
    if (world > std::max(n, 1)) throw std::invalid_argument("ras plan: more ranks than rows");
    Plan P;
    P.n = n;
    P.rank = rank;
    P.world = world;
    P.overlap = overlap;
    const Partition part = partition_graph(a, world);
    const std::vector<std::vector<int>> ext = extend_overlap(a, part, overlap);
    P.part_of = part.part_of;
    P.own = part.parts[rank];
    P.ext = ext[rank];

    // every rank's halo (a rank sends what the others' halos hold of its rows)
    std::vector<char> mark(static_cast<std::size_t>(n), 0);
    std::vector<std::vector<int>> halos(world);
    for (int p = 0; p < world; ++p) halos[p] = halo_of(a, part, ext[p], p, mark);
    P.halo = halos[rank];

    std::vector<int> pos_in_own(static_cast<std::size_t>(n), -1), loc(static_cast<std::size_t>(n), -1);
    for (int k = 0; k < P.n_own(); ++k) pos_in_own[P.own[k]] = loc[P.own[k]] = k;
    for (int k = 0; k < static_cast<int>(P.halo.size()); ++k) loc[P.halo[k]] = P.n_own() + k;

    P.send_offsets.assign(static_cast<std::size_t>(world) + 1, 0);
    P.recv_offsets.assign(static_cast<std::size_t>(world) + 1, 0);
    for (int p = 0; p < world; ++p) {
        if (p != rank)
            for (int r : halos[p])  // p's halo is ordered by owner: my rows are one ascending run
                if (part.part_of[r] == rank) P.send_idx.push_back(pos_in_own[r]);
        P.send_offsets[p + 1] = static_cast<int>(P.send_idx.size());
        int cnt = 0;
        for (int r : P.halo) cnt += part.part_of[r] == p;
        P.recv_offsets[p + 1] = P.recv_offsets[p] + cnt;
    }

    P.gather.resize(P.ext.size());
    P.out_index.resize(P.ext.size());
    for (std::size_t k = 0; k < P.ext.size(); ++k) {
        const int r = P.ext[k];
        P.gather[k] = loc[r];
        P.out_index[k] = part.part_of[r] == rank ? pos_in_own[r] : -1;
    }

    // local SpMV rows: A[own, :], storage order kept, columns renumbered
    CsrMatrix& L = P.a_local;
    L.n_rows = P.n_own();
    L.n_cols = P.n_loc();
    L.row_offsets.assign(static_cast<std::size_t>(L.n_rows) + 1, 0);
    for (int k = 0; k < L.n_rows; ++k) {
        const int r = P.own[k];
        L.row_offsets[k + 1] = L.row_offsets[k] + (a.row_offsets[r + 1] - a.row_offsets[r]);
    }
    L.col_indices.resize(static_cast<std::size_t>(L.row_offsets[L.n_rows]));
    L.values.resize(L.col_indices.size());
#pragma omp parallel for schedule(static)
    for (int k = 0; k < L.n_rows; ++k) {
        const int r = P.own[k];
        int d = L.row_offsets[k];
        for (int e = a.row_offsets[r]; e < a.row_offsets[r + 1]; ++e, ++d) {
            L.col_indices[d] = loc[a.col_indices[e]];
            L.values[d] = a.values[e];
        }
    }
    for (int c : L.col_indices)
        if (c < 0) throw std::logic_error("ras plan: SpMV column outside own + halo");
    return P;
}

}  // namespace hec::ras
