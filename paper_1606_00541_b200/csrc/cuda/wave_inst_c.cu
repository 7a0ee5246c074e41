// k_wave instantiations for sliced-ELL widths 7,8,10 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

 HEC_WAVE_INST(7) HEC_WAVE_INST(8) HEC_WAVE_INST(10)

void* wave_kernel_c(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
         HEC_PICK(7) HEC_PICK(8) HEC_PICK(10)
        default: return nullptr;
    }
}

}  // namespace hec::dev
