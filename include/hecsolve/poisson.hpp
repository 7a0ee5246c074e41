#pragma once
// Matrix generators for the benchmark configurations.
// gen_poisson7 is the drop-in for reference proj/include/hecsolve/poisson.hpp:7-10;
// the others are new (SURVEY.md §8(d) C2, C3, C5 define them).

#include <cstdint>
#include <vector>

#include "hecsolve/csr.hpp"

namespace hec {

// 7-point Laplacian, Dirichlet truncation, x-fastest numbering, diag 6.
CsrMatrix gen_poisson7(int nx, int ny, int nz);

// 27-point Laplacian, Dirichlet truncation, x-fastest numbering, diag 26,
// -1 to every existing neighbour in the 3x3x3 box.
CsrMatrix gen_poisson27(int nx, int ny, int nz);

// Heterogeneous 7-point finite-volume operator (SPE10-like contrast):
// cell permeability k = 10^(sigma (2u - 1)), u from mt19937_64(seed) in cell
// order; horizontal faces use k, vertical faces kz_ratio * k; interior faces
// carry the harmonic mean 2ab/(a+b); a boundary face adds the cell's own
// coefficient to the diagonal. sigma = 0, kz_ratio = 1 reproduces gen_poisson7.
CsrMatrix gen_reservoir7(int nx, int ny, int nz, double sigma = 3.0, double kz_ratio = 0.1,
                         std::uint64_t seed = 1606);

// Symmetric permutation B = P A P^T with B[perm[i], perm[j]] = A[i, j].
CsrMatrix permute_symmetric(const CsrMatrix& a, const std::vector<int>& perm);

// perm (original -> new) from std::shuffle with mt19937_64(seed).
std::vector<int> random_ordering(int n, std::uint64_t seed = 1606);

// Reverse Cuthill-McKee on the symmetrized pattern (original -> new).
std::vector<int> rcm_ordering(const CsrMatrix& a);

}  // namespace hec
