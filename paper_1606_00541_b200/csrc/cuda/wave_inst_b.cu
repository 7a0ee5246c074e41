// k_wave instantiations for sliced-ELL widths 4,5,6 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

 HEC_WAVE_INST(4) HEC_WAVE_INST(5) HEC_WAVE_INST(6)

void* wave_kernel_b(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
         HEC_PICK(4) HEC_PICK(5) HEC_PICK(6)
        default: return nullptr;
    }
}

}  // namespace hec::dev
