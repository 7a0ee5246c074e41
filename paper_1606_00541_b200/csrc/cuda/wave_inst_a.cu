// k_wave instantiations for sliced-ELL widths 1,2,3 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

void* wave_kernel_a(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
        case 1: return wave_pick<1>(group, groups, rpl, trace);
        case 2: return wave_pick<2>(group, groups, rpl, trace);
        case 3: return wave_pick<3>(group, groups, rpl, trace);
        default: return nullptr;
    }
}

}  // namespace hec::dev
