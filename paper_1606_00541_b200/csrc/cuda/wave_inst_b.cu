// k_wave instantiations for sliced-ELL widths 4,5,6 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

void* wave_kernel_b(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
        case 4: return wave_pick<4>(group, groups, rpl, trace);
        case 5: return wave_pick<5>(group, groups, rpl, trace);
        case 6: return wave_pick<6>(group, groups, rpl, trace);
        default: return nullptr;
    }
}

}  // namespace hec::dev
