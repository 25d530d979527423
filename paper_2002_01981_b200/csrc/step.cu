// step.cu -- the fused IFCM step (the hot path) for sm_100a.
//
// One launch = one Jacobi IFCM iteration (Alg. 2 steps 6-8,
// PAPER:179-181) for P states at once (grid.z = state).  Per voxel i and
// cluster j, from the previous memberships (R7):
//   Eq. 6  g_ik = |x_i - x_k|
//   Eq. 5  H_ij = sum_k u_kj g_ik / sum_k g_ik  0 if all g = 0 (R3)
//   Eq. 7  F_ij = sum_k u_kj^2 q2_ik / sum_k q2_ik  q2 per R1
//   Eq. 4  d2_ij = (x_i - c_j)^2 max(1 - lam H - xi F, 1e-9)  (R4)
//   Eq. 2  u_ij  = w_ij / sum_k w_ik, w = d2^{-1/(m-1)}       (R5)
//   Eq. 3 / Eq. 1 partial sums: sum u^m x, sum u^m, J, max|du|
// over the 26-neighbourhood of Eq. 9 (R2).
//
// Data layout: x fp32 [nz][ny][pitch]; U fp32 AoS-C4 [state][nz][ny][nx][4].
// CTA = 32 x 16 voxels per plane (4 warps, 4 y-rows per thread), marching
// kTZ planes in z through a 4-stage shared-memory ring filled by cp.async
// (zero-filled outside the volume, so out-of-bounds neighbours contribute 0
// to every numerator).  Because every U row sums to 1, the Eq. 5
// denominator is recovered as G_i = sum_j Hn_ij = sum_k g_ik sum_j u_kj, which
// automatically excludes out-of-bounds neighbours; the Eq. 7 denominator is a
// closed form of the in-bounds neighbour counts per offset class.
#include <cuda_runtime.h>

#include "pifcm_internal.cuh"

namespace pifcm {

__device__ __forceinline__ float rcp_approx(float v) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Per-voxel epilogue shared by the stencil and pointwise kernels: Eq. 4 with
// the given H, F; Eq. 2; accumulation of the Eq. 3 / Eq. 1 partial sums.
template <int C, bool M2>
__device__ __forceinline__ float4 membership(float xv, const float (&c)[kMaxC],
                                             const float (&a)[kMaxC], float m, float inv_m1,
                                             float (&num)[kMaxC], float (&den)[kMaxC],
                                             float &Jacc) {
    float d2[C];
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const float d = xv - c[j];
        d2[j] = d * d * a[j];                               // Eq. 4 (a already floored, R4)
    }
    float u[kMaxC] = {0.f, 0.f, 0.f, 0.f};
    int jz = C;
#pragma unroll
    for (int j = C - 1; j >= 0; --j)
        if (d2[j] == 0.0f) jz = j;
    float Ji;
    if (jz < C) {  // R5: zero distance -> crisp row at the lowest such j
#pragma unroll
        for (int j = 0; j < C; ++j) u[j] = (j == jz) ? 1.0f : 0.0f;
        Ji = 0.0f;
    } else {
        float w[C], S = 0.0f;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            w[j] = M2 ? rcp_approx(d2[j]) : exp2f(-log2f(d2[j]) * inv_m1);
            S += w[j];
        }
        const float invS = rcp_approx(S);
#pragma unroll
        for (int j = 0; j < C; ++j) u[j] = w[j] * invS;      // Eq. 2
        // Eq. 1 per voxel: sum_j u^m d2 = S^{1-m} (closed form of Eq. 2's u)
        Ji = M2 ? invS : exp2f((1.0f - m) * log2f(S));
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const float um = M2 ? u[j] * u[j] : (u[j] > 0.f ? exp2f(m * log2f(u[j])) : 0.f);
        num[j] = fmaf(um, xv, num[j]);  // Eq. 3 numerator
        den[j] += um;                   // Eq. 3 denominator
    }
    Jacc += Ji;
    return make_float4(u[0], u[1], u[2], u[3]);
}

// Attraction factor a_j = 1 - lam H_ij - xi F_ij (Eq. 4) re-evaluated in fp64
// directly from the definitions (Eq. 5-8: G = sum of in-bounds g, literal
// per-neighbour q2 weights) for a voxel whose fp32 factor fell in the
// ill-conditioned band near 0.  There d2_ij (and so u_ij) is proportional to
// a_j, so fp32 rounding of H and F (~1e-7 absolute) would be amplified by
// 1/a_j; fp64 keeps the step within the parity tolerance.
__device__ __noinline__ void attraction_fp64(const float4 *__restrict__ sU0, const float *__restrict__ sX0,
                                             int stage_stride, int sm, int sc, int sp, int row, int col,
                                             float xr, int gx, int gy, int z, int nx, int ny, int nz,
                                             double lam, double xi, float w2, float w3, int C, float *a_out) {
    double G = 0.0, Qs = 0.0, Hn[kMaxC] = {0.0, 0.0, 0.0, 0.0}, Fn[kMaxC] = {0.0, 0.0, 0.0, 0.0};
    for (int dz = -1; dz <= 1; ++dz) {
        const int s = dz < 0 ? sm : (dz == 0 ? sc : sp);
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (dx == 0 && dy == 0 && dz == 0) continue;
                if (gx + dx < 0 || gx + dx >= nx || gy + dy < 0 || gy + dy >= ny || z + dz < 0 ||
                    z + dz >= nz)
                    continue;
                const int e = s * stage_stride + (row + dy) * kSX + (col + dx);
                const float4 u = sU0[e];
                const double g = fabs((double)xr - (double)sX0[e]);
                const int n = (dx != 0) + (dy != 0) + (dz != 0);
                const double q2 = n == 1 ? 1.0 : (n == 2 ? (double)w2 : (double)w3);
                const double uk[4] = {u.x, u.y, u.z, u.w};
                G += g;
                Qs += q2;
                for (int j = 0; j < C; ++j) {
                    Hn[j] += uk[j] * g;
                    Fn[j] += uk[j] * uk[j] * q2;
                }
            }
    }
    for (int j = 0; j < C; ++j) {
        const double H = G > 0.0 ? Hn[j] / G : 0.0;
        const double F = Qs > 0.0 ? Fn[j] / Qs : 0.0;
        const double a = __dadd_rn(__dadd_rn(1.0, -__dmul_rn(lam, H)), -__dmul_rn(xi, F));
        a_out[j] = (float)fmax(a, (double)kAFloor);
    }
}

// Reduce the per-thread partial sums of the CTA into one fp64 record
// (fixed order: xor-shuffle tree in each warp, then warps in index order).
template <int NW>
__device__ __forceinline__ void block_partials(const float (&num)[kMaxC], const float (&den)[kMaxC],
                                               float Jacc, float duacc, double *out) {
    __shared__ double red[NW][kNR];
    double v[kNR];
#pragma unroll
    for (int j = 0; j < kMaxC; ++j) { v[j] = num[j]; v[kMaxC + j] = den[j]; }
    v[2 * kMaxC] = Jacc;
    v[2 * kMaxC + 1] = duacc;
#pragma unroll
    for (int r = 0; r < kNR; ++r) {
        double t = v[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double q = __shfl_xor_sync(0xffffffffu, t, o);
            t = (r == kNR - 1) ? fmax(t, q) : t + q;
        }
        v[r] = t;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < kNR; ++r) red[warp][r] = v[r];
    }
    __syncthreads();
    if (threadIdx.x < kNR) {
        const int r = threadIdx.x;
        double t = red[0][r];
        for (int w = 1; w < NW; ++w) t = (r == kNR - 1) ? fmax(t, red[w][r]) : t + red[w][r];
        out[r] = t;
    }
}

// ----------------------------------------------------------------------------
// Stencil step (lambda, xi arbitrary): the hot kernel.
template <int C, bool M2>
__global__ void __launch_bounds__(kStepThreads, 4) k_step_stencil(const StepArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4(*sU)[kSY][kSX] = reinterpret_cast<float4(*)[kSY][kSX]>(smem_raw);
    float(*sX)[kSY][kSX] =
        reinterpret_cast<float(*)[kSY][kSX]>(smem_raw + sizeof(float4) * kStages * kSY * kSX);

    const int p = blockIdx.z;
    if (a.stop && *a.stop) return;
    if (a.stats && a.stats[4 * p + 3] != 0.0) return;

    const int tile = blockIdx.x;
    const int x0 = (tile % a.tiles_x) * kTX;
    const int y0 = (tile / a.tiles_x) * kTY;
    const int zb = blockIdx.y * kTZ;
    const int ze = min(zb + kTZ, a.nz);
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;

    const long long plane = (long long)a.nx * a.ny;
    const float4 *Uin = a.U_in + (long long)(a.in_idx ? a.in_idx[p] : p) * a.nvox;
    float4 *Uout = a.U_out + (long long)(a.out_idx ? a.out_idx[p] : p) * a.nvox;

    float c[kMaxC];
#pragma unroll
    for (int j = 0; j < kMaxC; ++j) c[j] = a.centers[4 * p + j];
    const float lam = (float)a.lam_xi[2 * p], xi = (float)a.lam_xi[2 * p + 1];
    // Eq. 7 class weights: q2 for 1, 2, 3 non-zero offsets (R1)
    const float w1 = 1.0f, w2 = a.q_mode == 0 ? 4.0f : 2.0f, w3 = a.q_mode == 0 ? 9.0f : 3.0f;

    auto load_plane = [&](int z) {
        const int s = (z + kStages) & (kStages - 1);
        const bool zin = (z >= 0) && (z < a.nz);
        for (int e = tid; e < kSY * kSX; e += kStepThreads) {
            const int yy = e / kSX, xx = e - yy * kSX;
            const int gy = y0 - 1 + yy, gx = x0 - 1 + xx;
            const bool in = zin && gy >= 0 && gy < a.ny && gx >= 0 && gx < a.nx;
            const long long vi = in ? ((long long)z * plane + (long long)gy * a.nx + gx) : 0;
            cp_async16(&sU[s][yy][xx], Uin + vi, in);
            const long long xo = in ? ((long long)z * a.ny + gy) * a.pitch + gx : 0;
            cp_async4(&sX[s][yy][xx], a.x + xo, in);
        }
    };

    float num[kMaxC] = {0.f, 0.f, 0.f, 0.f}, den[kMaxC] = {0.f, 0.f, 0.f, 0.f};
    float Jacc = 0.f, duacc = 0.f;

    load_plane(zb - 1);
    load_plane(zb);
    load_plane(zb + 1);
    cp_async_commit();

    for (int z = zb; z < ze; ++z) {
        if (z + 2 <= ze) load_plane(z + 2);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();

        const int sm = (z - 1 + kStages) & (kStages - 1);
        const int sc = z & (kStages - 1);
        const int sp = (z + 1) & (kStages - 1);

        float xr[kRY];
#pragma unroll
        for (int r = 0; r < kRY; ++r) xr[r] = sX[sc][ty * kRY + 1 + r][tx + 1];

        float hn[kRY][C], fa[kRY][3][C];
#pragma unroll
        for (int r = 0; r < kRY; ++r)
#pragma unroll
            for (int j = 0; j < C; ++j) {
                hn[r][j] = 0.f;
                fa[r][0][j] = 0.f; fa[r][1][j] = 0.f; fa[r][2][j] = 0.f;
            }

#pragma unroll
        for (int dz = -1; dz <= 1; ++dz) {
            const int s = dz < 0 ? sm : (dz == 0 ? sc : sp);
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
#pragma unroll
                for (int t = 0; t < kRY + 2; ++t) {
                    const float4 uk4 = sU[s][ty * kRY + t][tx + 1 + dx];
                    const float xk = sX[s][ty * kRY + t][tx + 1 + dx];
                    const float uk[4] = {uk4.x, uk4.y, uk4.z, uk4.w};
#pragma unroll
                    for (int r = 0; r < kRY; ++r) {
                        const int dy = t - 1 - r;
                        if (dy < -1 || dy > 1) continue;
                        if (dx == 0 && dy == 0 && dz == 0) continue;  // Eq. 9: k != i
                        const int ncls = (dx != 0) + (dy != 0) + (dz != 0);
                        const float g = fabsf(xr[r] - xk);         // Eq. 6
#pragma unroll
                        for (int j = 0; j < C; ++j) {
                            hn[r][j] = fmaf(uk[j], g, hn[r][j]);          // Eq. 5 numerator
                            fa[r][ncls - 1][j] = fmaf(uk[j], uk[j], fa[r][ncls - 1][j]);  // Eq. 7
                        }
                    }
                }
            }
        }

        // Eq. 7 denominator from the in-bounds neighbour counts per class.
        const int gx = x0 + tx;
        const int px = (gx > 0) + (gx < a.nx - 1);
        const int pz = (z > 0) + (z < a.nz - 1);
#pragma unroll
        for (int r = 0; r < kRY; ++r) {
            const int gy = y0 + ty * kRY + r;
            if (gx >= a.nx || gy >= a.ny) continue;
            const int py = (gy > 0) + (gy < a.ny - 1);
            const float Qs = w1 * (float)(px + py + pz) + w2 * (float)(px * py + py * pz + pz * px) +
                             w3 * (float)(px * py * pz);
            const float invQ = Qs > 0.f ? 1.0f / Qs : 0.f;
            float G = 0.f;
#pragma unroll
            for (int j = 0; j < C; ++j) G += hn[r][j];  // = sum_k g_ik (rows of U sum to 1)
            const float invG = G > 0.f ? rcp_approx(G) : 0.f;  // R3
            float av[kMaxC] = {1.f, 1.f, 1.f, 1.f};
            bool band = false;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const float H = hn[r][j] * invG;                                           // Eq. 5
                const float F = fmaf(w3, fa[r][2][j], fmaf(w2, fa[r][1][j], w1 * fa[r][0][j])) * invQ;  // Eq. 7
                const float a1 = fmaf(-lam, H, fmaf(-xi, F, 1.0f));                      // Eq. 4 factor
                band |= (a1 > -kBandLo) && (a1 < kBandHi);
                av[j] = fmaxf(a1, kAFloor);                                              // R4
            }
            if (band && (lam > 0.f || xi > 0.f))
                attraction_fp64(&sU[0][0][0], &sX[0][0][0], kSY * kSX, sm, sc, sp, ty * kRY + 1 + r, tx + 1,
                                xr[r], gx, gy, z, a.nx, a.ny, a.nz, a.lam_xi[2 * p], a.lam_xi[2 * p + 1], w2, w3,
                                C, av);
            const float4 un = membership<C, M2>(xr[r], c, av, a.m, a.inv_m1, num, den, Jacc);
            const float4 uo = sU[sc][ty * kRY + 1 + r][tx + 1];
            duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                       fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
            Uout[(long long)z * plane + (long long)gy * a.nx + gx] = un;
        }
        __syncthreads();
    }
    cp_async_wait<0>();

    const int blk = blockIdx.x + gridDim.x * blockIdx.y;
    block_partials<kWarpsY>(num, den, Jacc, duacc, a.partials + ((long long)p * a.nblk + blk) * kNR);
}

// ----------------------------------------------------------------------------
// Pointwise step for lambda = xi = 0 (plain FCM, Alg. 2 step 5):
// Eq. 4 reduces to (x_i - c_j)^2, no neighbourhood is read.
template <int C, bool M2>
__global__ void __launch_bounds__(kPwThreads) k_step_pointwise(const StepArgs a) {
    const int p = blockIdx.y;
    if (a.stop && *a.stop) return;
    if (a.stats && a.stats[4 * p + 3] != 0.0) return;
    const float4 *Uin = a.U_in + (long long)(a.in_idx ? a.in_idx[p] : p) * a.nvox;
    float4 *Uout = a.U_out + (long long)(a.out_idx ? a.out_idx[p] : p) * a.nvox;
    float c[kMaxC];
#pragma unroll
    for (int j = 0; j < kMaxC; ++j) c[j] = a.centers[4 * p + j];
    const float av[kMaxC] = {1.f, 1.f, 1.f, 1.f};  // lambda = xi = 0: Eq. 4 factor is 1
    float num[kMaxC] = {0.f, 0.f, 0.f, 0.f}, den[kMaxC] = {0.f, 0.f, 0.f, 0.f};
    float Jacc = 0.f, duacc = a.first ? 1.0f : 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nvox; i += stride) {
        const int X = (int)(i % a.nx);
        const long long row = i / a.nx;  // = z*ny + y
        const float xv = a.x[row * a.pitch + X];
        const float4 un = membership<C, M2>(xv, c, av, a.m, a.inv_m1, num, den, Jacc);
        if (!a.first) {
            const float4 uo = Uin[i];
            duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                       fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
        }
        Uout[i] = un;
    }
    block_partials<kPwThreads / 32>(num, den, Jacc, duacc,
                                   a.partials + ((long long)p * a.nblk + blockIdx.x) * kNR);
}

// ----------------------------------------------------------------------------
static int pw_blocks(long long nvox) {
    long long b = (nvox + kPwThreads * 8 - 1) / (kPwThreads * 8);
    if (b > 148 * 8) b = 148 * 8;
    if (b < 1) b = 1;
    return (int)b;
}

int step_nblk(int nx, int ny, int nz, bool stencil) {
    if (!stencil) return pw_blocks((long long)nx * ny * nz);
    const int tx = (nx + kTX - 1) / kTX, ty = (ny + kTY - 1) / kTY, tz = (nz + kTZ - 1) / kTZ;
    return tx * ty * tz;
}

template <int C, bool M2>
static cudaError_t launch_t(const StepArgs &a, bool stencil, int P, cudaStream_t st) {
    if (stencil) {
        const size_t smem = (sizeof(float4) + sizeof(float)) * kStages * kSY * kSX;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_step_stencil<C, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            attr = true;
        }
        dim3 grid(a.tiles_x * a.tiles_y, a.zchunks, P);
        k_step_stencil<C, M2><<<grid, kStepThreads, smem, st>>>(a);
    } else {
        dim3 grid(a.nblk, P);
        k_step_pointwise<C, M2><<<grid, kPwThreads, 0, st>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_step(const StepArgs &a0, int C, bool stencil, int P, cudaStream_t st) {
    StepArgs a = a0;
    a.tiles_x = (a.nx + kTX - 1) / kTX;
    a.tiles_y = (a.ny + kTY - 1) / kTY;
    a.zchunks = (a.nz + kTZ - 1) / kTZ;
    a.nblk = step_nblk(a.nx, a.ny, a.nz, stencil);
    const bool m2 = (a.m == 2.0f);
    switch (C) {
        case 2: return m2 ? launch_t<2, true>(a, stencil, P, st) : launch_t<2, false>(a, stencil, P, st);
        case 3: return m2 ? launch_t<3, true>(a, stencil, P, st) : launch_t<3, false>(a, stencil, P, st);
        case 4: return m2 ? launch_t<4, true>(a, stencil, P, st) : launch_t<4, false>(a, stencil, P, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pifcm
