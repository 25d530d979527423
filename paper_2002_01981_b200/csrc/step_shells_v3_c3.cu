// step_shells_v3_c3.cu -- the v = 3 shell step for C = 3 (step_shells.cuh).
#include "step_shells.cuh"

namespace pifcm {
PIFCM_SHELLS_INSTANCE(3, 3)
}  // namespace pifcm
