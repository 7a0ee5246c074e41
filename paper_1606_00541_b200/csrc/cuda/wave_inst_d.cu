// k_wave instantiations for sliced-ELL widths 13,16 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

void* wave_kernel_d(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
        case 13: return wave_pick<13>(group, groups, rpl, trace);
        case 16: return wave_pick<16>(group, groups, rpl, trace);
        default: return nullptr;
    }
}

}  // namespace hec::dev
