// step_shells_v2_c4.cu -- the v = 2 shell step for C = 4 (step_shells.cuh).
#include "step_shells.cuh"

namespace pifcm {
PIFCM_SHELLS_INSTANCE(2, 4)
}  // namespace pifcm
