// Instantiation of k_wave for a set of sliced-ELL widths (one translation unit
// per width group, so the widths compile in parallel). Solver shapes
// (G warps per group x K groups, RPL rows per lane):
//   1x4x2   up to  64 rows per chunk (e.g. 27-point slabs)
//   1x8x2   up to  64 rows, deeper round robin
//   2x4x2   up to 128 rows
//   4x2x4   up to 512 rows (e.g. 7-point z-pencils)
//   4x4x4   up to 512 rows, deeper round robin
//   8x2x2   up to 512 rows, two rows per lane
#pragma once
#include "wave_kernel.cuh"

#define HEC_WAVE_INST4(WD, G, K, RP)                                \
    template __global__ void k_wave<WD, G, K, RP, false>(WaveArgs); \
    template __global__ void k_wave<WD, G, K, RP, true>(WaveArgs);
#define HEC_WAVE_INST(WD)                                                                                   \
    HEC_WAVE_INST4(WD, 1, 4, 2) HEC_WAVE_INST4(WD, 1, 8, 2) HEC_WAVE_INST4(WD, 2, 4, 2) HEC_WAVE_INST4(WD, 4, 2, 4) \
    HEC_WAVE_INST4(WD, 4, 4, 4) HEC_WAVE_INST4(WD, 8, 2, 2)
#define HEC_K(WD, G, K, RP) \
    (trace ? reinterpret_cast<void*>(&k_wave<WD, G, K, RP, true>) : reinterpret_cast<void*>(&k_wave<WD, G, K, RP, false>))
#define HEC_PICK(WD)                                                         \
    case WD:                                                                 \
        if (group == 1 && groups == 4 && rpl == 2) return HEC_K(WD, 1, 4, 2); \
        if (group == 1 && groups == 8 && rpl == 2) return HEC_K(WD, 1, 8, 2); \
        if (group == 2 && groups == 4 && rpl == 2) return HEC_K(WD, 2, 4, 2); \
        if (group == 4 && groups == 2 && rpl == 4) return HEC_K(WD, 4, 2, 4); \
        if (group == 4 && groups == 4 && rpl == 4) return HEC_K(WD, 4, 4, 4); \
        if (group == 8 && groups == 2 && rpl == 2) return HEC_K(WD, 8, 2, 2); \
        return nullptr;
