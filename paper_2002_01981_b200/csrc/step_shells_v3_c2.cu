// step_shells_v3_c2.cu -- the v = 3 shell step for C = 2 (step_shells.cuh).
#include "step_shells.cuh"

namespace pifcm {
PIFCM_SHELLS_INSTANCE(3, 2)
}  // namespace pifcm
