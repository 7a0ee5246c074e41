#pragma once
// Restricted Additive Schwarz with one subdomain per GPU: the host plan of one
// rank (reference proj/src/precond.cpp:74-117 build_preconditioner(ras) and
// proj/src/partition.cpp:28-107, split by owner).
//
// Rank g owns part g of partition_graph(A, world) (ascending global rows) and
// keeps a local vector [own | halo]: the halo is ext_g u cols(A[own, :]) minus
// own, ordered by (owning rank, global row), so each peer's contribution is
// one contiguous segment. With overlap 1 on a symmetric pattern the RAS halo
// (ext_g \ own) and the SpMV halo coincide; otherwise the union serves both.

#include <vector>

#include "hecsolve/csr.hpp"

namespace hec::ras {

struct Plan {
    int n = 0, rank = 0, world = 1, overlap = 0;
    std::vector<int> part_of;                // global row -> owning rank
    std::vector<int> own;                    // ascending global rows owned here
    std::vector<int> ext;                    // ascending rows of the extended part (the local block)
    std::vector<int> halo;                   // global rows of the halo segment, by (owner, row)
    std::vector<int> send_offsets;           // [world + 1] into send_idx
    std::vector<int> send_idx;               // own positions each peer needs, in the peer's halo order
    std::vector<int> recv_offsets;           // [world + 1] halo segment of each peer
    std::vector<int> gather;                 // block row k -> local [own | halo] index of ext[k]
    std::vector<int> out_index;              // block row k -> own position, or -1 (restriction)
    CsrMatrix a_local;                       // A[own, :], columns renumbered to [own | halo], storage order kept

    int n_own() const { return static_cast<int>(own.size()); }
    int n_loc() const { return static_cast<int>(own.size() + halo.size()); }
};

// Deterministic on every rank from the global matrix (no communication).
Plan make_plan(const CsrMatrix& a, int world, int rank, int overlap);

}  // namespace hec::ras
