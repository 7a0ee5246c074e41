// k_wave instantiations for sliced-ELL widths 13,16 (see wave_inst.cuh).
#include "wave_inst.cuh"

namespace hec::dev {

 HEC_WAVE_INST(13) HEC_WAVE_INST(16)

void* wave_kernel_d(int width, int group, int groups, int rpl, bool trace) {
    switch (width) {
         HEC_PICK(13) HEC_PICK(16)
        default: return nullptr;
    }
}

}  // namespace hec::dev
