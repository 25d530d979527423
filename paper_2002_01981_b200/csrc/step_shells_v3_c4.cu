// step_shells_v3_c4.cu -- the v = 3 shell step for C = 4 (step_shells.cuh).
#include "step_shells.cuh"

namespace pifcm {
PIFCM_SHELLS_INSTANCE(3, 4)
}  // namespace pifcm
