// step_shells_v2_c3.cu -- the v = 2 shell step for C = 3 (step_shells.cuh).
#include "step_shells.cuh"

namespace pifcm {
PIFCM_SHELLS_INSTANCE(2, 3)
}  // namespace pifcm
