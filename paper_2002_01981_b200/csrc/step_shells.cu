// step_shells.cu -- dispatch of the v = 2, 3 shell step (NEXT-2; Eq. 9-10,
// PAPER:81-85) to its per-(v, C) instances (step_shells_v<V>_c<C>.cu).
#include "pifcm_internal.cuh"

namespace pifcm {

#define PIFCM_SHELLS_DECL(V_, C_) cudaError_t launch_shells_##V_##_##C_(const StepArgs &a, int P, cudaStream_t st);
PIFCM_SHELLS_DECL(2, 2)
PIFCM_SHELLS_DECL(2, 3)
PIFCM_SHELLS_DECL(2, 4)
PIFCM_SHELLS_DECL(3, 2)
PIFCM_SHELLS_DECL(3, 3)
PIFCM_SHELLS_DECL(3, 4)

// The decomposition fields of `a` (tiles, z-chunks, nblk) are set by launch_step.
cudaError_t launch_step_shells(const StepArgs &a, int C, int P, cudaStream_t st) {
    if (C < 2 || C > 4) return cudaErrorInvalidValue;
    if (a.v == 2) return C == 2 ? launch_shells_2_2(a, P, st) : C == 3 ? launch_shells_2_3(a, P, st) : launch_shells_2_4(a, P, st);
    if (a.v == 3) return C == 2 ? launch_shells_3_2(a, P, st) : C == 3 ? launch_shells_3_3(a, P, st) : launch_shells_3_4(a, P, st);
    return cudaErrorInvalidValue;
}

}  // namespace pifcm
