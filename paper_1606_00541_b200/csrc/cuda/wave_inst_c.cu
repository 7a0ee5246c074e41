// k_wave instantiations for sliced-ELL widths 7,8,10 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

void* wave_kernel_c(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
        case 7: return wave_pick<7>(group, groups, rpl, trace);
        case 8: return wave_pick<8>(group, groups, rpl, trace);
        case 10: return wave_pick<10>(group, groups, rpl, trace);
        default: return nullptr;
    }
}

}  // namespace hec::dev
