// k_wave instantiations for sliced-ELL widths 1,2,3 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

 HEC_WAVE_INST(1) HEC_WAVE_INST(2) HEC_WAVE_INST(3)

void* wave_kernel_a(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
         HEC_PICK(1) HEC_PICK(2) HEC_PICK(3)
        default: return nullptr;
    }
}

}  // namespace hec::dev
