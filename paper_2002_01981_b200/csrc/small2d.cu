// small2d.cu -- many IFCM iterations of a small 2D image in one launch (the
// latency-bound config C1: a 32 x 32 slice, 20 iterations).
//
// One CTA per state holds the whole haloed image in shared memory (x and two
// membership buffers) and runs the Jacobi iterations back to back: Eq. 5-8 over
// the 8-neighbourhood of Eq. 9 (nz = 1), Eq. 4, Eq. 2 (the stencil kernels'
// epilogue: memb_compute, with the fp64 re-evaluation of ill-conditioned
// voxels), then the Eq. 3 centres and the Eq. 1 cost from a
// fixed-order block reduction in fp64 -- no grid-wide dependency, so no
// launch per iteration (pifcm_iterate at C1: ~26 us per iteration as one
// launch each, host-bound).
#include <cuda_runtime.h>

#include "pifcm_internal.cuh"
#include "step_common.cuh"

namespace pifcm {

constexpr int kS2Threads = 512;
constexpr int kS2Warps = kS2Threads / 32;

// Eq. 4 factors of one voxel from the definitions in fp64 (Eq. 5-8, R1, R3, R4).
template <int C>
__device__ __forceinline__ float4 factors_fp64_2d(const float4 *sU, const float *sx, int W, int X, int Y, int nx,
                                                  int ny, double lam, double xi, double w2) {
    double G = 0.0, Q = 0.0, hn[kMaxC] = {0.0, 0.0, 0.0, 0.0}, fn[kMaxC] = {0.0, 0.0, 0.0, 0.0};
    const double xi0 = (double)sx[(Y + 1) * W + X + 1];
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            if (dx == 0 && dy == 0) continue;
            if (X + dx < 0 || X + dx >= nx || Y + dy < 0 || Y + dy >= ny) continue;
            const int o = (Y + 1 + dy) * W + X + 1 + dx;
            const double g = fabs(xi0 - (double)sx[o]);                 // Eq. 6
            const double q2 = (dx != 0 && dy != 0) ? w2 : 1.0;           // Eq. 8, R1
            const float4 u = sU[o];
            const double uk[4] = {u.x, u.y, u.z, u.w};
            G += g;
            Q += q2;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                hn[j] += uk[j] * g;
                fn[j] += uk[j] * uk[j] * q2;
            }
        }
    float out[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const double H = G > 0.0 ? hn[j] / G : 0.0;  // Eq. 5, R3
        const double F = Q > 0.0 ? fn[j] / Q : 0.0;  // Eq. 7
        const double av = __dadd_rn(__dadd_rn(1.0, -__dmul_rn(lam, H)), -__dmul_rn(xi, F));  // Eq. 4
        out[j] = (float)fmax(av, (double)kAFloor);  // R4
    }
    return make_float4(out[0], out[1], out[2], out[3]);
}

template <int C, bool M2>
__global__ void __launch_bounds__(kS2Threads) k_iterate_small2d(const float *x, int nx, int ny, int pitch,
                                                                 const float4 *U_in, float4 *U_out, long long nvox,
                                                                 float *centers, const double *lam_xi, int iters,
                                                                 float eps, float m, float inv_m1, int q_mode,
                                                                 double *stats, int *status) {
    constexpr int NP = (C + 1) / 2;
    extern __shared__ __align__(16) unsigned char sm[];
    const int W = nx + 2, H2 = ny + 2;  // haloed extent
    float4 *sA = reinterpret_cast<float4 *>(sm);
    float4 *sB = sA + (size_t)W * H2;
    float *sx = reinterpret_cast<float *>(sB + (size_t)W * H2);
    __shared__ double red[kS2Warps][kNR];
    __shared__ float s_c[kMaxC];
    __shared__ int s_stop;
    const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = nx * ny;
    // load the state and x with zero halos (out-of-bounds neighbours contribute 0)
    for (int i = tid; i < W * H2; i += kS2Threads) {
        const int Y = i / W - 1, X = i % W - 1;
        const bool in = X >= 0 && X < nx && Y >= 0 && Y < ny;
        sA[i] = in ? U_in[(long long)p * nvox + (long long)Y * nx + X] : make_float4(0.f, 0.f, 0.f, 0.f);
        sB[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        sx[i] = in ? x[(long long)Y * pitch + X] : 0.f;
    }
    if (tid < kMaxC) s_c[tid] = centers[4 * p + tid];
    if (tid == 0) s_stop = 0;
    const double lamd = lam_xi[2 * p], xid = lam_xi[2 * p + 1];
    const float lam = (float)lamd, xi = (float)xid;
    const float w2 = q_mode == 0 ? 4.0f : 2.0f;
    __syncthreads();
    float4 *cur = sA, *nxt = sB;
    int t;
    double J = 0.0, du = 0.0;
    for (t = 1; t <= iters; ++t) {
        const float2 c2[2] = {make_float2(s_c[0], s_c[1]), make_float2(s_c[2], s_c[3])};
        float2 num2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float2 den2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float Jacc = 0.f, duacc = 0.f;
        for (int v = tid; v < n; v += kS2Threads) {
            const int Y = v / nx, X = v - Y * nx;
            const int o = (Y + 1) * W + X + 1;
            const float xv = sx[o];
            float G = 0.f;
            float hn[kMaxC] = {0.f, 0.f, 0.f, 0.f}, fe[kMaxC] = {0.f, 0.f, 0.f, 0.f},
                  fk[kMaxC] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (dx == 0 && dy == 0) continue;            // Eq. 9: k != i
                    const int ok = o + dy * W + dx;
                    const float g = fabsf(xv - sx[ok]);          // Eq. 6
                    const float4 u = cur[ok];
                    const float uk[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                    for (int j = 0; j < C; ++j) {
                        hn[j] = fmaf(uk[j], g, hn[j]);           // Eq. 5 numerator
                        if (dx != 0 && dy != 0) fk[j] = fmaf(uk[j], uk[j], fk[j]);  // Eq. 7: corners
                        else fe[j] = fmaf(uk[j], uk[j], fe[j]);                     // faces
                    }
                }
#pragma unroll
            for (int j = 0; j < C; ++j) G += hn[j];  // = sum_k g_ik (rows of U sum to 1)
            const int px = (X > 0) + (X < nx - 1), py = (Y > 0) + (Y < ny - 1);
            const float Qs = (float)(px + py) + w2 * (float)(px * py);  // Eq. 7 denominator (2D)
            const float invQ = Qs > 0.f ? 1.0f / Qs : 0.f;
            const float invG = G > 0.f ? 1.0f / G : 0.f;  // R3
            float a4[4] = {1.f, 1.f, 1.f, 1.f}, ar4[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const float Hj = hn[j] * invG;                   // Eq. 5
                const float Fj = fmaf(fk[j], w2, fe[j]) * invQ;  // Eq. 7
                ar4[j] = fmaf(Hj, -lam, fmaf(Fj, -xi, 1.f));     // Eq. 4
                a4[j] = fmaxf(ar4[j], kAFloor);                  // R4
            }
            float2 A[2] = {make_float2(a4[0], a4[1]), make_float2(a4[2], a4[3])};
            const float2 Ar[2] = {make_float2(ar4[0], ar4[1]), make_float2(ar4[2], ar4[3])};
            Memb mb = memb_compute<C, M2>(xv, c2, A, m, inv_m1, Ar);
            float4 un;
            if (!(mb.K <= kKMax)) {  // ill-conditioned: the factors from the definitions in fp64
                const float4 f = factors_fp64_2d<C>(cur, sx, W, X, Y, nx, ny, lamd, xid, (double)w2);
                const float2 Af[2] = {make_float2(f.x, f.y), make_float2(f.z, f.w)};
                un = membership2<C, M2>(xv, c2, Af, m, inv_m1, num2, den2, Jacc);
            } else {
                memb_accumulate<C, M2>(mb, xv, m, num2, den2, Jacc);
                un = make_float4(mb.u[0], mb.u[1], mb.u[2], mb.u[3]);
            }
            const float4 uo = cur[o];
            duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                       fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
            nxt[o] = un;
        }
        (void)NP;
        // fixed-order fp64 block reduction: xor trees in the warps, warps in order
        double vr[kNR] = {num2[0].x, num2[0].y, num2[1].x, num2[1].y, den2[0].x, den2[0].y, den2[1].x, den2[1].y,
                          Jacc, duacc};
#pragma unroll
        for (int r = 0; r < kNR; ++r)
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) {
                const double q = __shfl_xor_sync(0xffffffffu, vr[r], o2);
                vr[r] = (r == kNR - 1) ? fmax(vr[r], q) : vr[r] + q;
            }
        if (lane == 0)
#pragma unroll
            for (int r = 0; r < kNR; ++r) red[warp][r] = vr[r];
        __syncthreads();
        if (tid == 0) {
            double s[kNR];
            for (int r = 0; r < kNR; ++r) s[r] = red[0][r];
            for (int w = 1; w < kS2Warps; ++w)
                for (int r = 0; r < kNR; ++r) s[r] = (r == kNR - 1) ? fmax(s[r], red[w][r]) : s[r] + red[w][r];
            for (int j = 0; j < C; ++j)
                if (s[kMaxC + j] >= kDenEps) s_c[j] = (float)(s[j] / s[kMaxC + j]);  // Eq. 3, R9
            J = s[2 * kMaxC];
            du = s[kNR - 1];
            s_stop = (eps > 0.f && du < (double)eps) ? 1 : 0;
            if (!isfinite(J) && status) atomicExch(status, (int)PIFCM_ENUMERIC);
        }
        __syncthreads();
        float4 *tmp = cur; cur = nxt; nxt = tmp;
        if (s_stop) break;
    }
    const int done = t > iters ? iters : t;
    for (int v = tid; v < n; v += kS2Threads) {
        const int Y = v / nx, X = v - Y * nx;
        U_out[(long long)p * nvox + v] = cur[(Y + 1) * W + X + 1];
    }
    if (tid < kMaxC) centers[4 * p + tid] = s_c[tid];
    if (tid == 0 && stats) {
        stats[4 * p + 0] = J;
        stats[4 * p + 1] = du;
        stats[4 * p + 2] = (double)done;
        stats[4 * p + 3] = s_stop ? 1.0 : 0.0;
    }
}

size_t small2d_smem(int nx, int ny) { return (size_t)(nx + 2) * (ny + 2) * (2 * 16 + 4); }

cudaError_t launch_iterate_small2d(const float *x, int nx, int ny, int pitch, const float4 *U_in, float4 *U_out,
                                   float *centers, const double *lam_xi, int P, int iters, float eps, float m,
                                   int q_mode, int C, double *stats, int *status, cudaStream_t st) {
    const size_t smem = small2d_smem(nx, ny);
    const long long nvox = (long long)nx * ny;
    const float inv_m1 = 1.0f / (m - 1.0f);
    const bool m2 = (m == 2.0f);
#define PIFCM_S2(CC, MM)                                                                                        \
    do {                                                                                                        \
        cudaError_t e = cudaFuncSetAttribute(k_iterate_small2d<CC, MM>,                                         \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
        if (e != cudaSuccess) return e;                                                                         \
        k_iterate_small2d<CC, MM><<<P, kS2Threads, smem, st>>>(x, nx, ny, pitch, U_in, U_out, nvox, centers,   \
                                                               lam_xi, iters, eps, m, inv_m1, q_mode, stats,    \
                                                               status);                                         \
    } while (0)
    switch (C) {
        case 2: if (m2) PIFCM_S2(2, true); else PIFCM_S2(2, false); break;
        case 3: if (m2) PIFCM_S2(3, true); else PIFCM_S2(3, false); break;
        case 4: if (m2) PIFCM_S2(4, true); else PIFCM_S2(4, false); break;
        default: return cudaErrorInvalidValue;
    }
#undef PIFCM_S2
    return cudaGetLastError();
}

}  // namespace pifcm
