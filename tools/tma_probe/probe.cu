// Standalone probe of the TMA boxes used by k_step_stencil (debug aid).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int c3, int c4, int bytes, float *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
        if (RANK == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su(sm)), "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(su(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(sm)), "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}" ::"r"(su(&bar)) : "memory");
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float *>(sm)[i];
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const int nx = 40, ny = 37, nz = 19, pitch = 40;
    float *x, *U, *out;
    cudaMalloc(&x, 4ull * pitch * ny * nz);
    cudaMalloc(&U, 16ull * nx * ny * nz);
    cudaMalloc(&out, 1 << 20);
    cudaMemset(x, 0, 4ull * pitch * ny * nz);
    CUtensorMap mX, mU;
    const cuuint64_t dx[3] = {nx, ny, nz};
    const cuuint64_t sx[2] = {4ull * pitch, 4ull * pitch * ny};
    const cuuint32_t bx[3] = {36, 18, 1};
    const cuuint32_t e[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&mX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dx, sx, bx, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode X: %d\n", (int)r);
    const cuuint64_t du[5] = {4, nx, ny, nz, 1};
    const cuuint64_t sus[4] = {16, 16ull * nx, 16ull * nx * ny, 16ull * nx * ny * nz};
    const cuuint32_t bu[5] = {4, 34, 18, 1, 1};
    r = enc(&mU, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, U, du, sus, bu, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode U: %d\n", (int)r);
    int c0s[4] = {0, -4, 4, -1};
    for (int ci = 0; ci < 4; ++ci) {
        k<3><<<1, 128, 16384>>>(mX, c0s[ci], -1, 5, 0, 0, 2592, out);
        printf("3d c0=%d: %s\n", c0s[ci], cudaGetErrorString(cudaDeviceSynchronize()));
        if (cudaGetLastError() != cudaSuccess) break;
    }
    return 0;
}
