// fitness.cu -- the ANCHORED and LEADER fitness modes.
//
// In both modes every particle of a generation is evaluated from ONE shared
// state S (ANCHORED: the start (U0, c0); LEADER: S_t, which follows the gbest's
// evaluation, R22).  The neighbourhood terms H (Eq. 5) and F (Eq. 7) of S do
// not depend on (lambda, xi), so the stencil runs once per state (the H, F
// pass of k_step_stencil) and a particle's fitness -- the J of its step, Eq. 1
// with the previous centres (R8) -- is a pointwise function of x, H, F:
//   a_j = max(1 - lambda H_j - xi F_j, 1e-9)             (Eq. 4, R4)
//   d2_j = (x - c_j)^2 a_j                                 (Eq. 4)
//   J_i = (sum_j d2_j^{-1/(m-1)})^{1-m}                    (Eq. 1 with Eq. 2's u)
// which k_eval_shared evaluates for all particles of a voxel at once: lanes
// are particles, the voxel data (36 B) is staged in shared memory and read as
// a broadcast, so per voxel it is read once for the whole swarm.
#include <cuda_runtime.h>
#include <math.h>

#include "pifcm_internal.cuh"

namespace pifcm {

constexpr int kEvThreads = 256;           // 8 warps
constexpr int kEvWarps = kEvThreads / 32;
constexpr int kEvChunk = 256;             // voxels staged per block iteration

__device__ __forceinline__ float rcp_fast(float v) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

template <int C, bool M2>
__global__ void __launch_bounds__(kEvThreads) k_eval_shared(const float *__restrict__ x, int nx, int ny,
                                                            long long nvox, int pitch,
                                                            const float4 *__restrict__ hf,
                                                            const float *__restrict__ centers,
                                                            const double *__restrict__ pos, int P, float m,
                                                            double *__restrict__ partials) {
    __shared__ float sx[kEvChunk];
    __shared__ float4 sH[kEvChunk], sF[kEvChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int groups = (P + 31) / 32;
    float c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = centers[j];
    const float inv_m1 = 1.0f / (m - 1.0f);
    // this lane's particles: p = lane + 32 g
    constexpr int kMaxG = 32;  // P <= 1024
    double acc[kMaxG / 8];     // at most 4 groups per lane held in registers (P <= 128 fast path)
    float lam[kMaxG / 8], xi[kMaxG / 8];
    const int gl = groups < kMaxG / 8 ? groups : kMaxG / 8;
#pragma unroll
    for (int g = 0; g < kMaxG / 8; ++g) {
        acc[g] = 0.0;
        const int p = lane + 32 * g;
        lam[g] = (g < gl && p < P) ? (float)pos[2 * p] : 0.f;
        xi[g] = (g < gl && p < P) ? (float)pos[2 * p + 1] : 0.f;
    }
    for (long long base = (long long)blockIdx.x * kEvChunk; base < nvox; base += (long long)gridDim.x * kEvChunk) {
        __syncthreads();
        {
            const long long i = base + threadIdx.x;
            if (i < nvox) {
                const unsigned ui = (unsigned)i, row = ui / (unsigned)nx;  // nvox < 2^31
                sx[threadIdx.x] = x[(long long)row * pitch + (ui - row * (unsigned)nx)];
                sH[threadIdx.x] = hf[2 * i];
                sF[threadIdx.x] = hf[2 * i + 1];
            }
        }
        __syncthreads();
        const int n = (int)min((long long)kEvChunk, nvox - base);
#pragma unroll
        for (int g = 0; g < kMaxG / 8; ++g) {
            if (g >= gl) break;
            float part = 0.f;
            for (int v = warp; v < n; v += kEvWarps) {
                const float xv = sx[v];
                const float4 H = sH[v], F = sF[v];
                const float hh[4] = {H.x, H.y, H.z, H.w}, ff[4] = {F.x, F.y, F.z, F.w};
                float d2[4];
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    const float aj = fmaxf(fmaf(-lam[g], hh[j], fmaf(-xi[g], ff[j], 1.0f)), kAFloor);  // Eq. 4
                    const float dx = xv - c[j];
                    d2[j] = dx * dx * aj;
                }
                float Ji;
                if (M2) {
                    // J_i = 1 / sum_j 1/d2_j as one quotient of products (one MUFU
                    // instead of C + 1): prod_j d2_j / sum_j prod_{k != j} d2_k
                    float num, den;
                    if (C == 2) {
                        num = d2[0] * d2[1];
                        den = d2[0] + d2[1];
                    } else if (C == 3) {
                        const float p01 = d2[0] * d2[1];
                        num = p01 * d2[2];
                        den = fmaf(d2[0] + d2[1], d2[2], p01);
                    } else {
                        const float p01 = d2[0] * d2[1], p23 = d2[2] * d2[3];
                        num = p01 * p23;
                        den = fmaf(p01, d2[2] + d2[3], p23 * (d2[0] + d2[1]));
                    }
                    Ji = num * rcp_fast(den);
                    if (!(num >= 1e-30f) || !(den < 1e30f)) {  // tiny / zero distances (R5): the sum form
                        float S = 0.f;
#pragma unroll
                        for (int j = 0; j < C; ++j) S += rcp_fast(d2[j]);  // d2 = 0 -> +inf
                        Ji = rcp_fast(S);                                  // S = inf -> 0
                    }
                } else {
                    float S = 0.f;
#pragma unroll
                    for (int j = 0; j < C; ++j) S += exp2f(-log2f(d2[j]) * inv_m1);
                    Ji = exp2f((1.0f - m) * log2f(S));  // J_i = S^{1-m}
                }
                part += Ji;
            }
            acc[g] += (double)part;
        }
    }
    // per-warp partials [block][warp][P] (fixed order, summed by k_fit_sum)
    double *out = partials + ((long long)blockIdx.x * kEvWarps + warp) * P;
#pragma unroll
    for (int g = 0; g < kMaxG / 8; ++g) {
        const int p = lane + 32 * g;
        if (g < gl && p < P) out[p] = acc[g];
    }
}

int eval_shared_parts(long long nvox, int P) {
    (void)P;
    long long blocks = (nvox + kEvChunk - 1) / kEvChunk;
    if (blocks > 148LL * 8) blocks = 148LL * 8;
    if (blocks < 1) blocks = 1;
    return (int)blocks * kEvWarps;
}

cudaError_t launch_eval_shared(const float *x, int nx, int ny, int nz, int pitch, const float4 *hf,
                               const float *centers, const double *pos, int P, int C, float m, double *partials,
                               int *nparts, cudaStream_t st) {
    if (P > 128) return cudaErrorInvalidValue;  // 4 lane groups held in registers
    const long long nvox = (long long)nx * ny * nz;
    const int parts = eval_shared_parts(nvox, P);
    *nparts = parts;
    const int blocks = parts / kEvWarps;
    const bool m2 = (m == 2.0f);
#define PIFCM_EV(CC)                                                                                    \
    (m2 ? (k_eval_shared<CC, true><<<blocks, kEvThreads, 0, st>>>(x, nx, ny, nvox, pitch, hf, centers, pos, \
                                                                  P, m, partials), 0)                  \
        : (k_eval_shared<CC, false><<<blocks, kEvThreads, 0, st>>>(x, nx, ny, nvox, pitch, hf, centers, pos, \
                                                                   P, m, partials), 0))
    switch (C) {
        case 2: PIFCM_EV(2); break;
        case 3: PIFCM_EV(3); break;
        case 4: PIFCM_EV(4); break;
        default: return cudaErrorInvalidValue;
    }
#undef PIFCM_EV
    return cudaGetLastError();
}

// fitness[p] = fixed-order sum of the per-warp partials (one block per particle).
constexpr int kFsThreads = 256;
__global__ void __launch_bounds__(kFsThreads) k_fit_sum(const double *partials, int nparts, int P, double *fitness,
                                                        int *status) {
    __shared__ double red[kFsThreads];
    const int p = blockIdx.x;
    double v = 0.0;
    for (int k = threadIdx.x; k < nparts; k += kFsThreads) v += partials[(long long)k * P + p];
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = kFsThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        fitness[p] = red[0];
        if (!isfinite(red[0]) && status) atomicExch(status, (int)PIFCM_ENUMERIC);
    }
}

cudaError_t launch_fit_sum(const double *partials, int nparts, int P, double *fitness, int *status,
                           cudaStream_t st) {
    k_fit_sum<<<P, kFsThreads, 0, st>>>(partials, nparts, P, fitness, status);
    return cudaGetLastError();
}

// Before the snapshot / advance step of a generation: the step runs at the
// gbest particle's evaluation position of this generation, from the shared
// centres.  ANCHORED: only when the gbest improved (the step is guarded by
// hdr[kHNotImproved]); the snapshot centres start as the shared start's.
__global__ void k_mode_pre(SwarmDev s, const float *shared_c, double *lamxi, int mode) {
    const int g = s.hdr[kHGbest];
    if (g < 0) return;
    if (mode == PIFCM_FIT_ANCHORED && !s.hdr[kHImproved]) return;
    lamxi[0] = s.evalpos[2 * g];
    lamxi[1] = s.evalpos[2 * g + 1];
    if (mode == PIFCM_FIT_ANCHORED)
        for (int j = 0; j < kMaxC; ++j) s.gbest_c[j] = shared_c[j];
}
cudaError_t launch_mode_pre(SwarmDev s, const float *shared_c, double *lamxi, int mode, cudaStream_t st) {
    k_mode_pre<<<1, 1, 0, st>>>(s, shared_c, lamxi, mode);
    return cudaGetLastError();
}

// LEADER, after the advance S_t -> S_{t+1} (slot nxt[0], centres updated in
// place): S_{t+1} becomes the shared state; on an improvement it is also the
// gbest snapshot (its slot was pinned by the update kernel).
__global__ void k_leader_post(SwarmDev s, const float *shared_c) {
    s.cur[0] = s.nxt[0];
    if (s.hdr[kHImproved])
        for (int j = 0; j < kMaxC; ++j) s.gbest_c[j] = shared_c[j];
}
cudaError_t launch_leader_post(SwarmDev s, const float *shared_c, cudaStream_t st) {
    k_leader_post<<<1, 1, 0, st>>>(s, shared_c);
    return cudaGetLastError();
}

__global__ void k_set_hdr(int *hdr, int idx, int value) { hdr[idx] = value; }
cudaError_t launch_set_hdr(int *hdr, int idx, int value, cudaStream_t st) {
    k_set_hdr<<<1, 1, 0, st>>>(hdr, idx, value);
    return cudaGetLastError();
}

}  // namespace pifcm
