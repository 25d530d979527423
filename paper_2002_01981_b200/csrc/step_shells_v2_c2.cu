// step_shells_v2_c2.cu -- the v = 2 shell step for C = 2 (step_shells.cuh).
#include "step_shells.cuh"

namespace pifcm {
PIFCM_SHELLS_INSTANCE(2, 2)
}  // namespace pifcm
