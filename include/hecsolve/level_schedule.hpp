#pragma once
// Level-set analysis for lower-triangular patterns (paper §3, Algorithm 1).
// Drop-in for reference proj/include/hecsolve/level_schedule.hpp:14-38.

#include <vector>

#include "hecsolve/csr.hpp"

namespace hec {

// level_of is 1-based and indexed by original row; rows are renumbered level by
// level (ascending original index inside a level): perm = original -> new,
// inv_perm = new -> original, level_starts[k] = first new row of level k+1.
struct LevelSchedule {
    int n = 0;
    int nlev = 0;
    std::vector<int> level_of;
    std::vector<int> perm;
    std::vector<int> inv_perm;
    std::vector<int> level_starts;
};

// level(i) = 1 + max level(j) over the strictly-lower columns j of row i.
// A column above the diagonal is std::invalid_argument.
std::vector<int> compute_levels(const CsrMatrix& l);

// Stable counting sort of the rows by level. Levels must be >= 1 and cover
// 1..nlev without holes (std::invalid_argument otherwise).
LevelSchedule build_schedule(const std::vector<int>& levels);

// Symmetric renumbering: (i, j) -> (perm[i], perm[j]), columns re-sorted.
CsrMatrix reorder_matrix(const CsrMatrix& l, const LevelSchedule& s);

// out[perm[i]] = v[i].
std::vector<double> permute_vector(const std::vector<double>& v, const std::vector<int>& perm);

}  // namespace hec
