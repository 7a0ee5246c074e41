// Instantiation of k_wave for a set of sliced-ELL widths (one translation unit
// per width group, so the widths compile in parallel). Solver shapes the
// planner chooses (G warps per group x K groups, RPL rows per lane):
//   2x4x1   up to  64 rows per chunk (e.g. 27-point slabs; one row per lane: 27-pt
//           128^3 ILU apply 0.946 -> 0.922 ms against 1x4x2)
//   4x4x1   up to 128 rows (7-pt 128^3 0.277 -> 0.264 ms against 2x4x2)
//   1x4x2, 2x4x2   the same capacities with two rows per lane
//   4x3x4   up to 512 rows, widths <= 4 only (7-point z-pencils: three groups,
//           one producer and two waiter warps)
//   8x2x2   up to 512 rows, widths <= 4 only (the register budget of 736
//           threads does not hold wider rows)
//   4x2x4   up to 512 rows, any width (widths >= 7 spill a few registers)
#pragma once
#include "wave_kernel.cuh"

namespace hec::dev {

template <int WD, int G, int K, int RP>
void* wave_ptr(bool trace) {
    return trace ? reinterpret_cast<void*>(&k_wave<WD, G, K, RP, true>)
                 : reinterpret_cast<void*>(&k_wave<WD, G, K, RP, false>);
}

// taking the addresses instantiates exactly the supported shapes of width WD
template <int WD>
void* wave_pick(int group, int groups, int rpl, bool trace) {
    if (group == 1 && groups == 4 && rpl == 2) return wave_ptr<WD, 1, 4, 2>(trace);
    if (group == 2 && groups == 4 && rpl == 2) return wave_ptr<WD, 2, 4, 2>(trace);
    if (group == 2 && groups == 4 && rpl == 1) return wave_ptr<WD, 2, 4, 1>(trace);
    if (group == 4 && groups == 4 && rpl == 1) return wave_ptr<WD, 4, 4, 1>(trace);
    if (group == 4 && groups == 2 && rpl == 4) return wave_ptr<WD, 4, 2, 4>(trace);
    if constexpr (WD <= 4) {
        if (group == 8 && groups == 2 && rpl == 2) return wave_ptr<WD, 8, 2, 2>(trace);
        if (group == 4 && groups == 3 && rpl == 4) return wave_ptr<WD, 4, 3, 4>(trace);
    }
    return nullptr;
}

}  // namespace hec::dev
