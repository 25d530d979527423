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
// a z-chunk through a kRing-stage (5) shared-memory ring of haloed planes
// filled by TMA (cp.async.bulk.tensor, one mbarrier per stage; boxes are
// zero-filled outside the volume, so out-of-bounds neighbours contribute 0
// to every numerator).  Because every U row sums to 1, the Eq. 5
// denominator is recovered as G_i = sum_j Hn_ij = sum_k g_ik sum_j u_kj, which
// automatically excludes out-of-bounds neighbours; the Eq. 7 denominator is a
// closed form of the in-bounds neighbour counts per offset class.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "pifcm_internal.cuh"
#include "step_common.cuh"

namespace pifcm {

// Shared-memory ring: kRing planes of the haloed U tile (float4) and of the
// intensity tile (float, rows padded to kSXP for 16-byte TMA boxes).
// TMA requires a 16-byte-aligned start of the innermost box dimension, so the
// intensity box starts at x0 - 4 (not x0 - 1) and is 40 floats wide; the
// thread's own column sits at kXOff = 4.
constexpr int kSXP = 40;
constexpr int kXOff = 4;
constexpr int kUStageBytes = kSY * kSX * 16;  // 9792
constexpr int kXStageBytes = kSY * kSXP * 4;  // 2592
constexpr int kUStagePad = (kUStageBytes + 127) / 128 * 128;
constexpr int kXStagePad = (kXStageBytes + 127) / 128 * 128;
#ifndef PIFCM_STEP_MINBLOCKS
#define PIFCM_STEP_MINBLOCKS 3
#endif
constexpr int kStepMinBlocks = PIFCM_STEP_MINBLOCKS;  // CTAs per SM the register budget targets
#ifndef PIFCM_RING
#define PIFCM_RING 5
#endif
constexpr int kRing = PIFCM_RING;  // planes in flight: z-1, z, z+1 in use, the rest prefetching
#ifndef PIFCM_STATE_Y
#define PIFCM_STATE_Y 1  // 3D step grid (tile, state, chunk) instead of (tile, chunk, state)
#endif
#ifndef PIFCM_SMEM_SLACK
#define PIFCM_SMEM_SLACK 128
#endif
constexpr int kStencilSmem = kRing * (kUStagePad + kXStagePad) + PIFCM_SMEM_SLACK;

// Warp-cooperative fp64 re-evaluation of the Eq. 4 factors of one voxel (the
// ill-conditioned band): lane k < 26 takes neighbour k of
// the 26-neighbourhood (Eq. 9), the per-neighbour terms of Eq. 5 / Eq. 7
// (G = sum of in-bounds g, Qs = sum of in-bounds q2, numerators) are summed
// across the warp in fp64, and every lane returns the floored factors.
template <int C>
__device__ __forceinline__ float4 attraction_coop(const float4 *Um, const float4 *Uc, const float4 *Up,
                                                  const float *Xm, const float *Xc, const float *Xp,
                                                  int row, int col, int gx, int gy, int z, int nx, int ny,
                                                  int nz, double lam, double xi, double w2, double w3) {
    const int lane = threadIdx.x & 31;
    const int idx = lane < 13 ? lane : lane + 1;  // skip the centre (idx 13)
    const int dz = idx / 9 - 1, dy = (idx / 3) % 3 - 1, dx = idx % 3 - 1;
    double v[2 + 2 * kMaxC];
#pragma unroll
    for (int i = 0; i < 2 + 2 * kMaxC; ++i) v[i] = 0.0;
    const bool inb = lane < 26 && gx + dx >= 0 && gx + dx < nx && gy + dy >= 0 && gy + dy < ny &&
                     z + dz >= 0 && z + dz < nz;
    if (inb) {
        const float4 *Us = dz < 0 ? Um : (dz == 0 ? Uc : Up);
        const float *Xs = dz < 0 ? Xm : (dz == 0 ? Xc : Xp);
        const float4 u = Us[(row + dy) * kSX + col + 1 + dx];
        const double xr = (double)Xc[row * kSXP + col + kXOff];
        const double g = fabs(xr - (double)Xs[(row + dy) * kSXP + col + kXOff + dx]);  // Eq. 6
        const int n = (dx != 0) + (dy != 0) + (dz != 0);
        const double q2 = n == 1 ? 1.0 : (n == 2 ? w2 : w3);                            // Eq. 8, R1
        const double uk[4] = {u.x, u.y, u.z, u.w};
        v[0] = g;
        v[1] = q2;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            v[2 + j] = uk[j] * g;                     // Eq. 5 numerator term
            v[2 + kMaxC + j] = uk[j] * uk[j] * q2;   // Eq. 7 numerator term
        }
    }
#pragma unroll
    for (int i = 0; i < 2 + 2 * kMaxC; ++i) {
        if (i >= 2 + C && i < 2 + kMaxC) continue;
        if (i >= 2 + kMaxC + C) continue;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
    float out[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const double H = v[0] > 0.0 ? v[2 + j] / v[0] : 0.0;          // Eq. 5, R3
        const double F = v[1] > 0.0 ? v[2 + kMaxC + j] / v[1] : 0.0;  // Eq. 7
        const double av = __dadd_rn(__dadd_rn(1.0, -__dmul_rn(lam, H)), -__dmul_rn(xi, F));  // Eq. 4
        out[j] = (float)fmax(av, (double)kAFloor);                   // R4
    }
    return make_float4(out[0], out[1], out[2], out[3]);
}

// ----------------------------------------------------------------------------
// In-plane parts of the Eq. 7 numerator for the thread's own rows.  The Eq. 7
// numerator Fn_ij = sum_k q2_ik u_kj^2 is a linear 3x3x3 stencil of v = u^2
// whose weight depends only on the offset class n = |dX|+|dY|+|dZ| (Eq. 8,
// R1: q2 = W(n), W(1) = 1, W(2) = w2, W(3) = w3, W(0) = 0 for k = i).  Per
// plane it therefore splits into two in-plane stencils:
//   S (the target's own plane):  W(1) E + W(2) K
//   R (a plane at dZ = +-1):     W(1) v(0,0) + W(2) E + W(3) K
// with E = edge sum v(+-1,0) + v(0,+-1) and K = corner sum v(+-1,+-1), and
//   Fn(z) = R(z-1) + S(z) + R(z+1).
// Here v(x-1) + v(x+1) (d) and v(x) (c) are formed per haloed row and the
// rows are combined with a 3-row sliding window.
// MODE 0: S, R <- the sums of this plane.  MODE 1 (steady state, plane z+1 of
// target plane z): Fn = Pc + R; Pc = Rc + S; Rc = R, row by row.
template <int NP, int MODE>
__device__ __forceinline__ void plane_SR(const float4 *Us, int ty, int tx, float2 w22, float2 w32,
                                         float2 (&S)[kRY][NP], float2 (&R)[kRY][NP],
                                         float2 (&Fn)[kRY][NP]) {
    float2 dwin[3][NP], cwin[3][NP];
#pragma unroll
    for (int t = 0; t < kRY + 2; ++t) {
        const int o = (ty * kRY + t) * kSX + tx + 1;
        const float4 ul = Us[o - 1], uc = Us[o], ur = Us[o + 1];
        const float2 l2[2] = {make_float2(ul.x, ul.y), make_float2(ul.z, ul.w)};
        const float2 c2[2] = {make_float2(uc.x, uc.y), make_float2(uc.z, uc.w)};
        const float2 r2[2] = {make_float2(ur.x, ur.y), make_float2(ur.z, ur.w)};
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int qq = (NP == 1) ? 0 : q;
            dwin[t % 3][q] = __ffma2_rn(l2[qq], l2[qq], __fmul2_rn(r2[qq], r2[qq]));
            cwin[t % 3][q] = __fmul2_rn(c2[qq], c2[qq]);
        }
        if (t >= 2) {
            const int r = t - 2;  // rows t-2, t-1, t = r, r+1, r+2 around target row r+1
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const float2 E = __fadd2_rn(dwin[(t - 1) % 3][q], __fadd2_rn(cwin[(t - 2) % 3][q], cwin[t % 3][q]));
                const float2 K = __fadd2_rn(dwin[(t - 2) % 3][q], dwin[t % 3][q]);
                const float2 Sv = __ffma2_rn(K, w22, E);
                const float2 Rv = __ffma2_rn(K, w32, __ffma2_rn(E, w22, cwin[(t - 1) % 3][q]));
                if (MODE == 0) {
                    S[r][q] = Sv;
                    R[r][q] = Rv;
                } else {  // S = Pc, R = Rc (carried)
                    Fn[r][q] = __fadd2_rn(S[r][q], Rv);
                    S[r][q] = __fadd2_rn(R[r][q], Sv);
                    R[r][q] = Rv;
                }
            }
        }
    }
}

// ----------------------------------------------------------------------------
// Stencil step (lambda, xi arbitrary): the hot kernel.
//   thread (tx, ty): x = x0 + tx, rows y0 + ty*kRY + r (r < kRY) of plane z.
//   Eq. 5: per plane the thread streams the 9 (dx, dz) columns of kRY+2
//   haloed rows from shared memory; each loaded neighbour row updates up to 3
//   of its voxels: g (Eq. 6) for two voxels per FADD2, one FFMA2 per cluster
//   pair for the numerator.  Eq. 7: the separable in-plane sums S, R of the
//   newest plane (plane_SR), carried across the z march.
//   Planes arrive by TMA into a kRing-stage ring (one full mbarrier per
//   stage); each warp counts its release of a stage in shared memory and the
//   last warp to release it refills it, so warps are not lock-stepped.
template <int C, bool M2, bool DU, bool HF>
__global__ void __launch_bounds__(kStepThreads, kStepMinBlocks)
    k_step_stencil(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
                   const StepArgs a) {
    constexpr int NP = (C + 1) / 2;  // cluster pairs (FFMA2 lanes)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *base = smem_raw;  // >= 16-byte aligned: enough for non-swizzled TMA boxes
    auto sUst = [&](int s) { return reinterpret_cast<float4 *>(base + s * kUStagePad); };
    auto sXst = [&](int s) { return reinterpret_cast<float *>(base + kRing * kUStagePad + s * kXStagePad); };
    __shared__ __align__(8) uint64_t full[kRing];
    __shared__ int released[kRing];

    // grid (tile, state, chunk): the states of one (tile, chunk) run side by
    // side, so the intensity planes they share are read from L2, not HBM
    const int p = PIFCM_STATE_Y ? blockIdx.y : blockIdx.z;
    const int chunk = PIFCM_STATE_Y ? blockIdx.z : blockIdx.y;
    if (a.stop && *a.stop) return;
    if (a.stats && a.stats[4 * p + 3] != 0.0) return;

    const int tile = blockIdx.x;
    const int x0 = (tile % a.tiles_x) * kTX;
    const int y0 = (tile / a.tiles_x) * kTY;
    const int zb = a.z_lo + chunk * a.tz;
    const int ze = min(zb + a.tz, a.z_lo + a.nz_t);
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    const int slot = a.in_idx ? a.in_idx[p] : p;

    if (tid == 0) {
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&full[s], 1);
            released[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // TMA of plane q (q may lie outside [0, nz): the box is zero-filled).  The
    // tensor maps are used through their kernel-parameter addresses.  A stage
    // is refilled (with plane q + kRing) by the last warp that releases it.
    const CUtensorMap *pmU = &tmU, *pmX = &tmX;
#define PIFCM_ISSUE_PLANE(q_)                                                        \
    do {                                                                             \
        const int l_ = (q_) - (zb - 1);                                              \
        const int s_ = l_ % kRing;                                                   \
        mbar_expect_tx(&full[s_], kUStageBytes + kXStageBytes);                      \
        tma_load_4d(sUst(s_), pmU, &full[s_], 4 * (x0 - 1), y0 - 1, (q_), slot);     \
        tma_load_3d(sXst(s_), pmX, &full[s_], x0 - kXOff, y0 - 1, (q_));            \
    } while (0)
    auto wait_plane = [&](int q) {
        const int l = q - (zb - 1);
        mbar_wait(&full[l % kRing], (l / kRing) & 1);
    };

    if (tid == 0) {
        for (int q = zb - 1; q <= min(zb + kRing - 2, ze); ++q) PIFCM_ISSUE_PLANE(q);
    }

    float4 *Uout = a.U_out + (long long)(a.out_idx ? a.out_idx[p] : p) * a.nvox;
    const long long plane = (long long)a.nx * a.ny;
    float2 c2[2];
    c2[0] = make_float2(a.centers[4 * p + 0], a.centers[4 * p + 1]);
    c2[1] = make_float2(a.centers[4 * p + 2], a.centers[4 * p + 3]);
    const float lam = (float)a.lam_xi[2 * p], xi = (float)a.lam_xi[2 * p + 1];
    const float w2 = a.q_mode == 0 ? 4.0f : 2.0f, w3 = a.q_mode == 0 ? 9.0f : 3.0f;  // Eq. 7 q2 (R1)
    const float2 w22 = make_float2(w2, w2), w32 = make_float2(w3, w3);
    const int gx = x0 + tx;
    const int px = (gx > 0) + (gx < a.nx - 1);
    // Eq. 7 denominator (closed form of the in-bounds neighbour counts per
    // class) for interior planes (pz = 2), per own row
    float invQi[kRY];
#pragma unroll
    for (int r = 0; r < kRY; ++r) {
        const int gy = y0 + ty * kRY + r;
        const int py = (gy > 0) + (gy < a.ny - 1);
        const float Qs = (float)(px + py + 2) + w2 * (float)(px * py + 2 * py + 2 * px) + w3 * (float)(px * py * 2);
        invQi[r] = 1.0f / Qs;
    }

    // rows of this thread that lie inside the volume, and their output row base
    unsigned vmask = 0u;
#pragma unroll
    for (int r = 0; r < kRY; ++r)
        if (gx < a.nx && y0 + ty * kRY + r < a.ny) vmask |= 1u << r;
    float4 *Urow = Uout + (long long)(y0 + ty * kRY) * a.nx + gx;

    float2 num2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float2 den2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float Jacc = 0.f, duacc = 0.f;

    // Eq. 7 carried sums: Pc = R(z-1) + S(z), Rc = R(z)
    float2 Pc[kRY][NP], Rc[kRY][NP];
    wait_plane(zb - 1);
    wait_plane(zb);
    {
        float2 S0[kRY][NP], R0[kRY][NP], S1[kRY][NP], R1[kRY][NP], dummy[kRY][NP];
        plane_SR<NP, 0>(sUst(0), ty, tx, w22, w32, S0, R0, dummy);  // plane zb-1 (local index 0)
        plane_SR<NP, 0>(sUst(1), ty, tx, w22, w32, S1, R1, dummy);  // plane zb
#pragma unroll
        for (int r = 0; r < kRY; ++r)
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                Pc[r][q] = __fadd2_rn(R0[r][q], S1[r][q]);
                Rc[r][q] = R1[r][q];
            }
    }

    for (int z = zb; z < ze; ++z) {
        wait_plane(z + 1);
        const int lz = z - (zb - 1);
        const int sm = (lz - 1) % kRing, sc = lz % kRing, sp = (lz + 1) % kRing;
        const float4 *Um = sUst(sm), *Uc = sUst(sc), *Up = sUst(sp);
        const float *Xm = sXst(sm), *Xc = sXst(sc), *Xp = sXst(sp);

        float xr[kRY];
#pragma unroll
        for (int r = 0; r < kRY; ++r) xr[r] = Xc[(ty * kRY + 1 + r) * kSXP + tx + kXOff];

        // ---- Eq. 5 numerators (and, on the z+1 plane, the Eq. 7 plane sums)
        float2 hn[kRY][NP];
#pragma unroll
        for (int r = 0; r < kRY; ++r)
#pragma unroll
            for (int q = 0; q < NP; ++q) hn[r][q] = make_float2(0.f, 0.f);
        // one loaded neighbour row (column dx, plane dz, haloed row t): g_ik
        // (Eq. 6) for the voxels it touches, two per FADD2, and the Eq. 5
        // numerators, one FFMA2 per cluster pair
        auto h_row = [&](const int dx, const int dz, const int t, const float4 uk4, const float xk) {
            const float2 u01 = make_float2(uk4.x, uk4.y), u23 = make_float2(uk4.z, uk4.w);
            float gv[kRY];
#pragma unroll
            for (int r = 0; r < kRY; r += 2) {
                const int dy0 = t - 1 - r, dy1 = t - 2 - r;
                const bool v0 = dy0 >= -1 && dy0 <= 1 && !(dx == 0 && dy0 == 0 && dz == 0);
                const bool v1 = dy1 >= -1 && dy1 <= 1 && !(dx == 0 && dy1 == 0 && dz == 0);
                if (v0 && v1) {
                    const float2 d = __fadd2_rn(make_float2(xr[r], xr[r + 1]), make_float2(-xk, -xk));
                    gv[r] = d.x;
                    gv[r + 1] = d.y;
                } else if (v0) {
                    gv[r] = xr[r] - xk;
                } else if (v1) {
                    gv[r + 1] = xr[r + 1] - xk;
                }
            }
#pragma unroll
            for (int r = 0; r < kRY; ++r) {
                const int dy = t - 1 - r;
                if (dy < -1 || dy > 1) continue;
                if (dx == 0 && dy == 0 && dz == 0) continue;  // Eq. 9: k != i
                const float g = fabsf(gv[r]);
                const float2 g2 = make_float2(g, g);
                hn[r][0] = __ffma2_rn(u01, g2, hn[r][0]);                 // Eq. 5 numerator
                if (NP > 1) hn[r][NP - 1] = __ffma2_rn(u23, g2, hn[r][NP - 1]);
            }
        };
#pragma unroll
        for (int dz = -1; dz <= 0; ++dz) {
            const float4 *Us = dz < 0 ? Um : Uc;
            const float *Xs = dz < 0 ? Xm : Xc;
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
                for (int t = 0; t < kRY + 2; ++t)
                    h_row(dx, dz, t, Us[(ty * kRY + t) * kSX + tx + 1 + dx],
                          Xs[(ty * kRY + t) * kSXP + tx + kXOff + dx]);
        }
        // plane z+1, row-major: the same loads feed Eq. 5 and the separable
        // Eq. 7 sums of plane_SR (Fn(z) = Pc + R(z+1); Pc = R(z) + S(z+1);
        // Rc = R(z+1)), so plane z+1 is read from shared memory once
        float2 Fn[kRY][NP];
        {
            float2 dwin[3][NP], cwin[3][NP];
#pragma unroll
            for (int t = 0; t < kRY + 2; ++t) {
                const int o = (ty * kRY + t) * kSX + tx + 1;
                const int ox = (ty * kRY + t) * kSXP + tx + kXOff;
                const float4 ul = Up[o - 1], uc = Up[o], ur = Up[o + 1];
                h_row(-1, 1, t, ul, Xp[ox - 1]);
                h_row(0, 1, t, uc, Xp[ox]);
                h_row(1, 1, t, ur, Xp[ox + 1]);
                const float2 l2[2] = {make_float2(ul.x, ul.y), make_float2(ul.z, ul.w)};
                const float2 cc[2] = {make_float2(uc.x, uc.y), make_float2(uc.z, uc.w)};
                const float2 r2[2] = {make_float2(ur.x, ur.y), make_float2(ur.z, ur.w)};
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    dwin[t % 3][q] = __ffma2_rn(l2[q], l2[q], __fmul2_rn(r2[q], r2[q]));
                    cwin[t % 3][q] = __fmul2_rn(cc[q], cc[q]);
                }
                if (t >= 2) {
                    const int r = t - 2;
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const float2 E = __fadd2_rn(dwin[(t - 1) % 3][q], __fadd2_rn(cwin[(t - 2) % 3][q], cwin[t % 3][q]));
                        const float2 K = __fadd2_rn(dwin[(t - 2) % 3][q], dwin[t % 3][q]);
                        const float2 Sv = __ffma2_rn(K, w22, E);
                        const float2 Rv = __ffma2_rn(K, w32, __ffma2_rn(E, w22, cwin[(t - 1) % 3][q]));
                        Fn[r][q] = __fadd2_rn(Pc[r][q], Rv);
                        Pc[r][q] = __fadd2_rn(Rc[r][q], Sv);
                        Rc[r][q] = Rv;
                    }
                }
            }
        }

        // ---- per-voxel epilogue: Eq. 5 / 7 ratios, Eq. 4, Eq. 2, partial sums
        float invQ[kRY];
        const int gz = z + a.goff;  // global plane (z-slab mode: z counts from the lower halo)
        const int pz = (gz > 0) + (gz < a.nz_g - 1);
        if (pz == 2) {
#pragma unroll
            for (int r = 0; r < kRY; ++r) invQ[r] = invQi[r];
        } else {  // first / last plane: fewer in-bounds neighbours (Eq. 7 denominator)
#pragma unroll
            for (int r = 0; r < kRY; ++r) {
                const int gy = y0 + ty * kRY + r;
                const int py = (gy > 0) + (gy < a.ny - 1);
                const float Qs = (float)(px + py + pz) + w2 * (float)(px * py + py * pz + pz * px) +
                                 w3 * (float)(px * py * pz);
                invQ[r] = Qs > 0.f ? 1.0f / Qs : 0.f;
            }
        }
        float4 *Uo = Urow + (long long)z * plane;  // this row's output (advanced by one image row per r)
        unsigned band_bits = 0u;
        if (!HF) {
            // the four rows' Eq. 4 / Eq. 2 without branches, then one warp
            // vote each for the rare paths (a zero distance, R5; a factor
            // small enough that the sensitivity K must be formed), then the
            // per-row partial sums and stores
            float u[kRY][4], Ji[kRY], S[kRY], Kr[kRY], d2v[kRY][4];
            float2 Arr[kRY][2];
            bool need_any = false;
#pragma unroll
            for (int r = 0; r < kRY; ++r) {
                float G = hn[r][0].x + hn[r][0].y;
                if (C > 2) G += hn[r][NP - 1].x;
                if (C > 3) G += hn[r][NP - 1].y;  // = sum_k g_ik (rows of U sum to 1)
                const float invG = G > 0.f ? rcp_approx(G) : 0.f;  // R3
                const float sl = -lam * invG, sx = -xi * invQ[r];  // Eq. 5 / 7 denominators folded
                const float2 x2 = make_float2(xr[r], xr[r]);
                float w[4] = {0.f, 0.f, 0.f, 0.f};
                float Sr = 0.f;
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    Arr[r][q] = __ffma2_rn(hn[r][q], make_float2(sl, sl),
                                           __ffma2_rn(Fn[r][q], make_float2(sx, sx), make_float2(1.f, 1.f)));  // Eq. 4
                    const float2 Aq = make_float2(fmaxf(Arr[r][q].x, kAFloor), fmaxf(Arr[r][q].y, kAFloor));  // R4
                    const float2 d = __fadd2_rn(x2, make_float2(-c2[q].x, -c2[q].y));
                    const float2 e = __fmul2_rn(__fmul2_rn(d, d), Aq);  // Eq. 4
                    d2v[r][2 * q] = e.x;
                    d2v[r][2 * q + 1] = e.y;
                }
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    w[j] = M2 ? rcp_approx(d2v[r][j]) : exp2f(-log2f(d2v[r][j]) * a.inv_m1);  // d2 = 0 -> +inf
                    Sr += w[j];
                }
                const float invS = rcp_approx(Sr);
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const float2 uu = __fmul2_rn(make_float2(w[2 * q], w[2 * q + 1]), make_float2(invS, invS));  // Eq. 2
                    u[r][2 * q] = uu.x;
                    u[r][2 * q + 1] = uu.y;
                }
                if (NP == 1) { u[r][2] = 0.f; u[r][3] = 0.f; }
                Ji[r] = M2 ? invS : exp2f((1.0f - a.m) * log2f(Sr));  // Eq. 1 per voxel: S^{1-m}
                S[r] = Sr;
                Kr[r] = 0.f;
                float amin = fminf(fabsf(Arr[r][0].x), fabsf(Arr[r][0].y));
                if (NP > 1) amin = fminf(amin, fminf(fabsf(Arr[r][NP - 1].x), fabsf(Arr[r][NP - 1].y)));
                // K <= (1 - 1/C) / min_j |a_j| (x 1/(m-1)): below kKMax the
                // voxel is not in the band (NaN factors fall through to K)
                need_any |= !(amin * kKMax >= 0.75f * (M2 ? 1.0f : a.inv_m1));
            }
            if (__any_sync(0xffffffffu, need_any)) {
#pragma unroll
                for (int r = 0; r < kRY; ++r) {
                    float Kp[2] = {0.f, 0.f};
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const float2 uu = make_float2(u[r][2 * q], u[r][2 * q + 1]);
                        const float2 ia = make_float2(rcp_approx(fabsf(Arr[r][q].x)), rcp_approx(fabsf(Arr[r][q].y)));
                        const float2 t = __fmul2_rn(__fmul2_rn(uu, __fadd2_rn(make_float2(1.f, 1.f), make_float2(-uu.x, -uu.y))), ia);
                        Kp[q] = t.x + ((2 * q + 1 < C) ? t.y : 0.f);
                    }
                    Kr[r] = M2 ? Kp[0] + Kp[1] : (Kp[0] + Kp[1]) * a.inv_m1;
                }
            }
            bool crisp_any = false;
#pragma unroll
            for (int r = 0; r < kRY; ++r) crisp_any |= !(S[r] < INFINITY);
            if (__any_sync(0xffffffffu, crisp_any)) {  // R5: a zero distance -> crisp row at the lowest such j
#pragma unroll
                for (int r = 0; r < kRY; ++r) {
                    if (S[r] < INFINITY) continue;
                    int jz = C - 1;
#pragma unroll
                    for (int j = C - 1; j >= 0; --j)
                        if (d2v[r][j] == 0.0f) jz = j;
#pragma unroll
                    for (int j = 0; j < 4; ++j) u[r][j] = (j == jz) ? 1.0f : 0.0f;
                    Ji[r] = 0.0f;
                    Kr[r] = 0.0f;
                }
            }
#pragma unroll
            for (int r = 0; r < kRY; ++r) {
                const bool valid = (vmask >> r) & 1u;
                const bool band = valid && !(Kr[r] <= kKMax);  // ill-conditioned: fp64 pass below
                band_bits |= band ? (1u << r) : 0u;
                const bool ok = valid && !band;
                const float4 un = make_float4(u[r][0], u[r][1], u[r][2], u[r][3]);
                if (ok) {
                    Memb mb;
#pragma unroll
                    for (int j = 0; j < 4; ++j) mb.u[j] = u[r][j];
                    mb.Ji = Ji[r];
                    mb.K = Kr[r];
                    memb_accumulate<C, M2>(mb, xr[r], a.m, num2, den2, Jacc);
                    if (DU) {
                        const float4 uo = Uc[(ty * kRY + 1 + r) * kSX + tx + 1];
                        duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                                   fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                    }
                    *Uo = un;
                }
                Uo += a.nx;
            }
        }
        if (HF) {  // particle-invariant H, F of this state (ANCHORED / LEADER fitness)
#pragma unroll
            for (int r = 0; r < kRY; ++r) {
                float G = hn[r][0].x + hn[r][0].y;
                if (C > 2) G += hn[r][NP - 1].x;
                if (C > 3) G += hn[r][NP - 1].y;  // = sum_k g_ik (rows of U sum to 1)
                const float invG = G > 0.f ? rcp_approx(G) : 0.f;  // R3
                float2 Hh[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                float2 Ff[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    Hh[q] = __fmul2_rn(hn[r][q], make_float2(invG, invG));        // Eq. 5
                    Ff[q] = __fmul2_rn(Fn[r][q], make_float2(invQ[r], invQ[r]));  // Eq. 7
                }
                if ((vmask >> r) & 1u) {
                    float4 *o = a.hf + 2 * ((long long)z * plane + (long long)(y0 + ty * kRY + r) * a.nx + gx);
                    o[0] = make_float4(Hh[0].x, Hh[0].y, Hh[1].x, Hh[1].y);
                    o[1] = make_float4(Ff[0].x, Ff[0].y, Ff[1].x, Ff[1].y);
                }
            }
        }

        // Ill-conditioned voxels of this warp, one at a time, all lanes together.
        unsigned lanes = __ballot_sync(0xffffffffu, band_bits != 0u);
        while (lanes) {
            const int L = __ffs(lanes) - 1;
            lanes &= lanes - 1;
            unsigned bits = __shfl_sync(0xffffffffu, band_bits, L);
            while (bits) {
                const int r = __ffs(bits) - 1;
                bits &= bits - 1;
                const int row = ty * kRY + 1 + r;
                const int gxL = x0 + L, gy = y0 + ty * kRY + r;
                const float4 a4 = attraction_coop<C>(Um, Uc, Up, Xm, Xc, Xp, row, L, gxL, gy, gz, a.nx, a.ny,
                                                     a.nz_g, a.lam_xi[2 * p], a.lam_xi[2 * p + 1], w2, w3);
                if (tx == L) {
                    const float2 A[2] = {make_float2(a4.x, a4.y), make_float2(a4.z, a4.w)};
                    const float xv = Xc[row * kSXP + L + kXOff];
                    const float4 un = membership2<C, M2>(xv, c2, A, a.m, a.inv_m1, num2, den2, Jacc);
                    if (DU) {
                        const float4 uo = Uc[row * kSX + L + 1];
                        duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                                   fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                    }
                    Uout[(long long)z * plane + (long long)gy * a.nx + gxL] = un;
                }
            }
        }
        // this warp no longer needs plane z-1; the last warp to release its
        // stage refills it with plane z-1+kRing
        __syncwarp();
        if (tx == 0) {
            const int old = atomicAdd(&released[sm], 1);
            if (old == kWarpsY - 1) {
                released[sm] = 0;
                if (z - 1 + kRing <= ze) PIFCM_ISSUE_PLANE(z - 1 + kRing);
            }
        }
    }
#undef PIFCM_ISSUE_PLANE

    if (HF) return;  // no reductions: H, F only
    float num[kMaxC] = {num2[0].x, num2[0].y, num2[1].x, num2[1].y};
    float den[kMaxC] = {den2[0].x, den2[0].y, den2[1].x, den2[1].y};
    const int blk = blockIdx.x + gridDim.x * chunk;  // record index: (tile, chunk), whatever the grid order
    block_partials<kWarpsY>(num, den, Jacc, duacc, a.partials + ((long long)p * a.nblk + blk) * kNR);
    // the ring is idle now: its shared memory is the finaliser's scratch
    // (no static 10 KB array, which would cost a CTA slot per SM)
    finalize_if_last<kStepThreads>(a, p, a.nblk, reinterpret_cast<double(*)[kNR]>(smem_raw));
}

// ----------------------------------------------------------------------------
// 2D step (nz = 1: the 8-neighbourhood of Eq. 9 in one plane -- the paper's
// Table 7 images, config C2).  The 3D kernel would stream two zero-filled
// neighbour planes through its ring and spend two thirds of its Eq. 5 work on
// them; here one TMA load brings the haloed tile, Eq. 5 runs over the three
// in-plane columns only and the Eq. 7 numerator is the in-plane sum S of
// plane_SR (faces W1 = 1, corners W2).  The epilogue is the 3D kernel's.
#ifndef PIFCM_2D_MINBLOCKS
#define PIFCM_2D_MINBLOCKS 5
#endif
// A CTA walks a column of kTYB2D tiles in y, the next tile's TMA load in
// flight while the current one is computed (two smem buffers).  One call =
// this CTA's tiles of one Jacobi step of state p, ending with its block
// record; `call` = how many earlier calls this CTA made (k_step_2d_loop's
// iteration): the two TMA buffers' mbarrier parities continue across calls.
template <int C, bool M2, bool DU>
__device__ __forceinline__ void step2d_tiles(const CUtensorMap *pmU, const CUtensorMap *pmX, const StepArgs &a,
                                             const int p, unsigned char *sbuf, uint64_t *bar, const int call) {
    constexpr int NP = (C + 1) / 2;
    // (stage pointers are formed from the __shared__ array at each use, so the
    // compiler keeps them in the shared window: LDS, not generic loads)
    auto sUb = [&](int b) { return reinterpret_cast<float4 *>(sbuf + b * kUStagePad); };
    auto sXb = [&](int b) { return reinterpret_cast<float *>(sbuf + 2 * kUStagePad + b * kXStagePad); };
    const int txi = blockIdx.x % a.tiles_x;
    const int ty0 = (blockIdx.x / a.tiles_x) * kTYB2D;
    const int ntile = min(kTYB2D, a.tiles_y - ty0);
    const int x0 = txi * kTX;
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    const int slot = a.in_idx ? a.in_idx[p] : p;
    auto issue = [&](int k) {
        const int b = k & 1, y0k = (ty0 + k) * kTY;
        mbar_expect_tx(&bar[b], kUStageBytes + kXStageBytes);
        tma_load_4d(sUb(b), pmU, &bar[b], 4 * (x0 - 1), y0k - 1, 0, slot);
        tma_load_3d(sXb(b), pmX, &bar[b], x0 - kXOff, y0k - 1, 0);
    };
    if (tid == 0) {
        issue(0);
        if (ntile > 1) issue(1);
    }
    float4 *Uout = a.U_out + (long long)(a.out_idx ? a.out_idx[p] : p) * a.nvox;
    float2 c2[2];
    // (L2 loads: in k_step_2d_loop another CTA finalised them this launch)
    c2[0] = make_float2(__ldcg(a.centers + 4 * p + 0), __ldcg(a.centers + 4 * p + 1));
    c2[1] = make_float2(__ldcg(a.centers + 4 * p + 2), __ldcg(a.centers + 4 * p + 3));
    const float lam = (float)a.lam_xi[2 * p], xi = (float)a.lam_xi[2 * p + 1];
    const float2 nlam2 = make_float2(-lam, -lam), nxi2 = make_float2(-xi, -xi);
    const float w2 = a.q_mode == 0 ? 4.0f : 2.0f, w3 = a.q_mode == 0 ? 9.0f : 3.0f;  // Eq. 7 q2 (R1)
    const float2 w22 = make_float2(w2, w2), w32 = make_float2(w3, w3);
    const int gx = x0 + tx;
    const int px = (gx > 0) + (gx < a.nx - 1);
    float2 num2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float2 den2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float Jacc = 0.f, duacc = 0.f;

#pragma unroll 1  // one copy of the tile body (an unrolled loop overflows the instruction cache)
    for (int k = 0; k < ntile; ++k) {
        const int b = k & 1;
        const float4 *sU = sUb(b);
        const float *sX = sXb(b);
        const int y0 = (ty0 + k) * kTY;
        float invQ[kRY];
        unsigned vmask = 0u;
#pragma unroll
        for (int r = 0; r < kRY; ++r) {
            const int gy = y0 + ty * kRY + r;
            const int py = (gy > 0) + (gy < a.ny - 1);
            const float Qs = (float)(px + py) + w2 * (float)(px * py);  // Eq. 7 denominator, pz = 0
            invQ[r] = Qs > 0.f ? 1.0f / Qs : 0.f;
            if (gx < a.nx && gy < a.ny) vmask |= 1u << r;
        }
        // buffer b is used (ntile + 1 - b) / 2 times per call
        mbar_wait(&bar[b], (unsigned)(call * ((ntile + 1 - b) / 2) + (k >> 1)) & 1u);

        float xr[kRY];
#pragma unroll
        for (int r = 0; r < kRY; ++r) xr[r] = sX[(ty * kRY + 1 + r) * kSXP + tx + kXOff];
        // Eq. 5 numerators over the 8 in-plane neighbours: every loaded row
        // updates up to 3 of the thread's voxels; g (Eq. 6) two voxels per FADD2
        float2 hn[kRY][NP];
#pragma unroll
        for (int r = 0; r < kRY; ++r)
#pragma unroll
            for (int q = 0; q < NP; ++q) hn[r][q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
            for (int t = 0; t < kRY + 2; ++t) {
                const float4 uk4 = sU[(ty * kRY + t) * kSX + tx + 1 + dx];
                const float xk = sX[(ty * kRY + t) * kSXP + tx + kXOff + dx];
                const float2 u01 = make_float2(uk4.x, uk4.y), u23 = make_float2(uk4.z, uk4.w);
                float gv[kRY];
#pragma unroll
                for (int r = 0; r < kRY; r += 2) {
                    const int dy0 = t - 1 - r, dy1 = t - 2 - r;
                    const bool v0 = dy0 >= -1 && dy0 <= 1 && !(dx == 0 && dy0 == 0);
                    const bool v1 = dy1 >= -1 && dy1 <= 1 && !(dx == 0 && dy1 == 0);
                    if (v0 && v1) {
                        const float2 d = __fadd2_rn(make_float2(xr[r], xr[r + 1]), make_float2(-xk, -xk));
                        gv[r] = d.x;
                        gv[r + 1] = d.y;
                    } else if (v0) {
                        gv[r] = xr[r] - xk;
                    } else if (v1) {
                        gv[r + 1] = xr[r + 1] - xk;
                    }
                }
#pragma unroll
                for (int r = 0; r < kRY; ++r) {
                    const int dy = t - 1 - r;
                    if (dy < -1 || dy > 1) continue;
                    if (dx == 0 && dy == 0) continue;  // Eq. 9: k != i
                    const float g = fabsf(gv[r]);
                    const float2 g2 = make_float2(g, g);
                    hn[r][0] = __ffma2_rn(u01, g2, hn[r][0]);
                    if (NP > 1) hn[r][NP - 1] = __ffma2_rn(u23, g2, hn[r][NP - 1]);
                }
            }
        // Eq. 7 numerator: the in-plane sum S = W1 E + W2 K of v = u^2
        float2 Fn[kRY][NP], Rd[kRY][NP], dummy[kRY][NP];
        plane_SR<NP, 0>(sU, ty, tx, w22, w32, Fn, Rd, dummy);

        float4 *Urow = Uout + (long long)(y0 + ty * kRY) * a.nx + gx;
        unsigned band_bits = 0u;
#pragma unroll
        for (int r = 0; r < kRY; ++r) {
            float G = hn[r][0].x + hn[r][0].y;
            if (C > 2) G += hn[r][NP - 1].x;
            if (C > 3) G += hn[r][NP - 1].y;  // = sum_k g_ik (rows of U sum to 1)
            const float invG = G > 0.f ? rcp_approx(G) : 0.f;  // R3
            float2 A[2], Ar[2];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const float2 H = __fmul2_rn(hn[r][q], make_float2(invG, invG));          // Eq. 5
                const float2 F = __fmul2_rn(Fn[r][q], make_float2(invQ[r], invQ[r]));    // Eq. 7
                Ar[q] = __ffma2_rn(H, nlam2, __ffma2_rn(F, nxi2, make_float2(1.f, 1.f))); // Eq. 4
                A[q].x = fmaxf(Ar[q].x, kAFloor);                                          // R4
                A[q].y = fmaxf(Ar[q].y, kAFloor);
            }
            if (NP == 1) { A[1] = make_float2(1.f, 1.f); Ar[1] = A[1]; }
            const Memb mb = memb_compute<C, M2>(xr[r], c2, A, a.m, a.inv_m1, Ar);
            const bool valid = (vmask >> r) & 1u;
            const bool band = valid && !(mb.K <= kKMax);  // ill-conditioned: fp64 pass below
            band_bits |= band ? (1u << r) : 0u;
            if (valid && !band) {
                memb_accumulate<C, M2>(mb, xr[r], a.m, num2, den2, Jacc);
                const float4 un = make_float4(mb.u[0], mb.u[1], mb.u[2], mb.u[3]);
                if (DU) {
                    const float4 uo = sU[(ty * kRY + 1 + r) * kSX + tx + 1];
                    duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                               fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                }
                Urow[(long long)r * a.nx] = un;
            }
        }
        // ill-conditioned voxels: the warp re-evaluates them in fp64 (nz = 1:
        // the out-of-plane neighbours are out of bounds and never read)
        unsigned lanes = __ballot_sync(0xffffffffu, band_bits != 0u);
        while (lanes) {
            const int L = __ffs(lanes) - 1;
            lanes &= lanes - 1;
            unsigned bits = __shfl_sync(0xffffffffu, band_bits, L);
            while (bits) {
                const int r = __ffs(bits) - 1;
                bits &= bits - 1;
                const int row = ty * kRY + 1 + r;
                const int gxL = x0 + L, gy = y0 + ty * kRY + r;
                const float4 a4 = attraction_coop<C>(sU, sU, sU, sX, sX, sX, row, L, gxL, gy, 0, a.nx, a.ny, 1,
                                                     a.lam_xi[2 * p], a.lam_xi[2 * p + 1], w2, w3);
                if (tx == L) {
                    const float2 A[2] = {make_float2(a4.x, a4.y), make_float2(a4.z, a4.w)};
                    const float xv = sX[row * kSXP + L + kXOff];
                    const float4 un = membership2<C, M2>(xv, c2, A, a.m, a.inv_m1, num2, den2, Jacc);
                    if (DU) {
                        const float4 uo = sU[row * kSX + L + 1];
                        duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                                   fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                    }
                    Uout[(long long)gy * a.nx + gxL] = un;
                }
            }
        }
        // every warp is done with buffer b: refill it with tile k + 2
        __syncthreads();
        if (tid == 0 && k + 2 < ntile) issue(k + 2);
    }
    float num[kMaxC] = {num2[0].x, num2[0].y, num2[1].x, num2[1].y};
    float den[kMaxC] = {den2[0].x, den2[0].y, den2[1].x, den2[1].y};
    block_partials<kWarpsY>(num, den, Jacc, duacc, a.partials + ((long long)p * a.nblk + blockIdx.x) * kNR);
}

template <int C, bool M2, bool DU>
__global__ void __launch_bounds__(kStepThreads, PIFCM_2D_MINBLOCKS)
    k_step_2d(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX, const StepArgs a) {
    // TMA destinations: 128-byte aligned stages (as the 3D ring)
    __shared__ __align__(128) unsigned char sbuf[2 * (kUStagePad + kXStagePad)];
    __shared__ __align__(8) uint64_t bar[2];
    const int p = blockIdx.z;
    if (a.stop && *a.stop) return;
    if (a.stats && a.stats[4 * p + 3] != 0.0) return;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    step2d_tiles<C, M2, DU>(&tmU, &tmX, a, p, sbuf, bar, 0);
    finalize_if_last<kStepThreads>(a, p, a.nblk);
}

// Grid-wide barrier of a cooperative launch (every CTA resident): arrival
// counter gbar[0], generation gbar[1] (both 0 before the launch; gbar[2] is
// k_step_2d_loop's finalisation release word).
__device__ __forceinline__ void grid_barrier(unsigned *gbar, unsigned nblocks, unsigned &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned target = gen + 1u;
        if (atomicAdd(&gbar[0], 1u) == nblocks - 1u) {
            gbar[0] = 0u;
            __threadfence();
            atomicExch(&gbar[1], target);
        } else {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gbar + 1) : "memory");
            } while (g < target);
        }
        __threadfence();
    }
    ++gen;
    __syncthreads();
}

// The final IFCM of one 2D state (nz = 1, P = 1) in one cooperative launch:
// `iters` Jacobi steps ping-ponging between UA (input of step 0) and UB, each
// followed by a grid barrier, the canonical finalisation by CTA 0 (the same
// fixed-order sum, thread count and Eq. 3 / Eq. 1 as the last-CTA finaliser
// of k_step_2d, so the results equal one launch per step bit for bit), a
// second barrier, and the convergence test (stats[3], max|du| < eps).  Saves
// the launch, ramp-up and tail of every step of a latency-bound small launch.
template <int C, bool M2>
__global__ void __launch_bounds__(kStepThreads, PIFCM_2D_MINBLOCKS)
    k_step_2d_loop(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmX, const StepArgs a, float4 *UA, float4 *UB, int iters,
                   unsigned *gbar) {
    __shared__ __align__(128) unsigned char sbuf[2 * (kUStagePad + kXStagePad)];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned gen = 0u;
    for (int t = 0; t < iters; ++t) {
        StepArgs at = a;
        at.U_out = (t & 1) ? UA : UB;
        // the previous step's states (generic stores) are read by TMA (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        step2d_tiles<C, M2, true>((t & 1) ? &tmB : &tmA, &tmX, at, 0, sbuf, bar, t);
        grid_barrier(gbar, gridDim.x, gen);
        // CTA 0 finalises; the others wait for its release word gbar[2]
        // (a broadcast, not a second all-CTA barrier)
        if (blockIdx.x == 0) {
            finalize_state<kStepThreads>(at, 0, a.nblk, reinterpret_cast<double(*)[kNR]>(sbuf));
            if (threadIdx.x == 0) {
                __threadfence();
                atomicExch(&gbar[2], (unsigned)(t + 1));
            }
        } else if (threadIdx.x == 0) {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gbar + 2) : "memory");
            } while (g < (unsigned)(t + 1));
            __threadfence();
        }
        __syncthreads();
        if (__ldcg(a.stats_out + 3) != 0.0) break;  // converged (eps): the last step's output is final
    }
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
    // grid-stride over voxels (coalesced); 32-bit index arithmetic (nvox < 2^31
    // is checked by the host)
    const unsigned nx = (unsigned)a.nx, nvox = (unsigned)a.nvox;
    const unsigned stride = gridDim.x * blockDim.x;
    // kPwILP voxels per thread per round, their loads issued before any use
    // (more bytes in flight per thread: the kernel is HBM-latency bound)
    constexpr int kPwILP = 4;
    for (unsigned i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < nvox; i0 += kPwILP * stride) {
        float xv[kPwILP];
        float4 uo[kPwILP];
#pragma unroll
        for (int k = 0; k < kPwILP; ++k) {
            const unsigned i = i0 + k * stride;
            if (i < nvox) {
                const unsigned row = i / nx;  // = z*ny + y
                xv[k] = __ldg(a.x + (size_t)row * a.pitch + (i - row * nx));
                if (!a.first) uo[k] = __ldcs(Uin + i);
            }
        }
#pragma unroll
        for (int k = 0; k < kPwILP; ++k) {
            const unsigned i = i0 + k * stride;
            if (i < nvox) {
                const float4 un = membership<C, M2>(xv[k], c, av, a.m, a.inv_m1, num, den, Jacc);
                if (!a.first)
                    duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo[k].x), fabsf(un.y - uo[k].y)),
                                               fmaxf(fabsf(un.z - uo[k].z), fabsf(un.w - uo[k].w))));
                __stcs(Uout + i, un);
            }
        }
    }
    block_partials<kPwThreads / 32>(num, den, Jacc, duacc,
                                   a.partials + ((long long)p * a.nblk + blockIdx.x) * kNR);
    finalize_if_last<kPwThreads>(a, p, a.nblk);
}

// ----------------------------------------------------------------------------
static int pw_blocks(long long nvox) {
    long long b = (nvox + kPwThreads * kPwSpan - 1) / (kPwThreads * kPwSpan);
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return (int)b;
}

// z-chunks of a stencil launch.  Depends on the volume only (not on the
// number of states), so the partial-sum decomposition -- and therefore every
// reduction result -- is the same whether a state is evaluated alone, in a
// batch, or on any rank of a particle-sharded run.  Chosen to fill whole
// waves of CTA slots (148 SMs x kStepMinBlocks) for a single state (the
// final IFCM), weighing the 2 halo planes each chunk re-reads; batched
// launches are many waves deep either way.
int step_zchunks(int nx, int ny, int nz, int P) {
    (void)P;
    const long long tiles = (long long)((nx + kTX - 1) / kTX) * ((ny + kTY - 1) / kTY);
    const long long slots = 148LL * kStepMinBlocks;
    const int zmax = (nz + kTZMin - 1) / kTZMin;
    int best = (nz + kTZ - 1) / kTZ;
    double best_eff = -1.0;
    for (int z = 1; z <= zmax; ++z) {
        const int tz = (nz + z - 1) / z;
        const int zz = (nz + tz - 1) / tz;  // chunks actually needed with tz planes each
        const long long ctas = tiles * zz;
        const long long waves = (ctas + slots - 1) / slots;
        const double eff = (double)ctas / (double)(waves * slots) * (double)tz / (double)(tz + 2);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = zz;
        }
    }
    return best;
}

// Planes per z-chunk of the canonical / z-slab decomposition: a function of
// the volume alone (never of the slab count), so the chunk records -- and with
// them centres and J -- are the same for any number of slabs.  Chosen like
// step_zchunks for one state on one GPU (wave fill x halo overhead), subject
// to at least 8 chunks (up to 8 slabs get work).
#ifndef PIFCM_HALO_COST
#define PIFCM_HALO_COST 2.0  // planes of work a chunk's halo and prologue cost (canonical chooser)
#endif
int slab_tz(int nx, int ny, int nz) {
    const long long tiles = (long long)((nx + kTX - 1) / kTX) * ((ny + kTY - 1) / kTY);
    const long long slots = 148LL * kStepMinBlocks;
    const int zmax = (nz + kTZMin - 1) / kTZMin;
    const int zmin = zmax < 8 ? zmax : 8;
    int best = (nz + zmin - 1) / zmin;
    double best_eff = -1.0;
    for (int z = zmin; z <= zmax; ++z) {
        const int tz = (nz + z - 1) / z;
        const int zz = (nz + tz - 1) / tz;
        if (zz < zmin) continue;
        const long long ctas = tiles * zz;
        const long long waves = (ctas + slots - 1) / slots;
        const double eff = (double)ctas / (double)(waves * slots) * (double)tz / ((double)tz + PIFCM_HALO_COST);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = tz;
        }
    }
    return best;
}

int step_nblk(int nx, int ny, int nz, bool stencil, int P) {
    if (!stencil) return pw_blocks((long long)nx * ny * nz);
    const int tx = (nx + kTX - 1) / kTX, ty = (ny + kTY - 1) / kTY;
    if (nz == 1) return tx * ((ty + kTYB2D - 1) / kTYB2D);  // k_step_2d: columns of kTYB2D tiles
    return tx * ty * step_zchunks(nx, ny, nz, P);
}

int step_nblk_max(int nx, int ny, int nz) {
    const int tx = (nx + kTX - 1) / kTX, ty = (ny + kTY - 1) / kTY;
    const int s = tx * ty * ((nz + kTZMin - 1) / kTZMin), q = pw_blocks((long long)nx * ny * nz);
    return s > q ? s : q;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// U states: 5-D (4 floats, x, y, z, state); x: 3-D (x, y, z) with pitched rows.
#ifndef PIFCM_U_L2_PROMOTION
#define PIFCM_U_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
static bool make_maps(const StepArgs &a, CUtensorMap *mU, CUtensorMap *mX) {
    auto enc = encode_fn();
    if (!enc) return false;
    // innermost dimension = whole AoS rows (4 * nx floats) so that every box
    // row is one contiguous 544-byte burst
    const cuuint64_t du[4] = {4ull * a.nx, (cuuint64_t)a.ny, (cuuint64_t)a.nz, (cuuint64_t)a.n_in_states};
    const cuuint64_t su[3] = {16ull * a.nx, 16ull * a.nx * a.ny, 16ull * (cuuint64_t)a.nvox};
    const cuuint32_t bu[4] = {4 * kSX, kSY, 1, 1};
    const cuuint32_t e5[5] = {1, 1, 1, 1, 1};
    if (enc(mU, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float4 *>(a.U_in), du, su, bu, e5,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, PIFCM_U_L2_PROMOTION,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const cuuint64_t dx[3] = {(cuuint64_t)a.nx, (cuuint64_t)a.ny, (cuuint64_t)a.nz};
    const cuuint64_t sx[2] = {4ull * a.pitch, 4ull * a.pitch * a.ny};
    const cuuint32_t bx[3] = {kSXP, kSY, 1};
    return enc(mX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(a.x), dx, sx, bx, e5,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C, bool M2, bool DU, bool HF = false>
static cudaError_t launch_stencil(const StepArgs &a, int P, cudaStream_t st) {
    // the dynamic shared-memory opt-in is per device: remember it per device
    static unsigned long long attr_set = 0ull;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    if (dev < 64 && !(attr_set & (1ull << dev))) {
        const cudaError_t e = cudaFuncSetAttribute(k_step_stencil<C, M2, DU, HF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   kStencilSmem);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << dev;
    }
    CUtensorMap mU, mX;
    if (!make_maps(a, &mU, &mX)) return cudaErrorInvalidValue;
    dim3 grid(a.tiles_x * a.tiles_y, PIFCM_STATE_Y ? P : a.zchunks, PIFCM_STATE_Y ? a.zchunks : P);
    k_step_stencil<C, M2, DU, HF><<<grid, kStepThreads, kStencilSmem, st>>>(mU, mX, a);
    return cudaGetLastError();
}

template <int C, bool M2, bool DU>
static cudaError_t launch_2d(const StepArgs &a, int P, cudaStream_t st) {
    CUtensorMap mU, mX;
    if (!make_maps(a, &mU, &mX)) return cudaErrorInvalidValue;
    dim3 grid(a.tiles_x * ((a.tiles_y + kTYB2D - 1) / kTYB2D), 1, P);
    k_step_2d<C, M2, DU><<<grid, kStepThreads, 0, st>>>(mU, mX, a);
    return cudaGetLastError();
}

template <int C, bool M2>
static cudaError_t launch_t(const StepArgs &a, bool stencil, int P, cudaStream_t st) {
    if (stencil && a.nz == 1 && a.nz_g == 1 && !a.hf)  // a plain 2D image (8-neighbourhood)
        return a.want_du ? launch_2d<C, M2, true>(a, P, st) : launch_2d<C, M2, false>(a, P, st);
    if (stencil) {
        if (a.hf) return M2 ? launch_stencil<C, true, false, true>(a, P, st) : cudaErrorInvalidValue;
        return a.want_du ? launch_stencil<C, M2, true>(a, P, st) : launch_stencil<C, M2, false>(a, P, st);
    }
    dim3 grid(a.nblk, P);
    k_step_pointwise<C, M2><<<grid, kPwThreads, 0, st>>>(a);
    return cudaGetLastError();
}

template <int C, bool M2>
static cudaError_t launch_2d_loop_t(const StepArgs &a, float4 *UA, float4 *UB, int iters, unsigned *gbar,
                                    cudaStream_t st, bool *used) {
    int dev = 0, nsm = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_2d_loop<C, M2>, kStepThreads, 0) !=
            cudaSuccess)
        return cudaErrorInvalidValue;
    const int grid = a.tiles_x * ((a.tiles_y + kTYB2D - 1) / kTYB2D);
    if (grid > per_sm * nsm) return cudaSuccess;  // not co-resident: the caller launches per step
    StepArgs aa = a, ab = a;
    aa.U_in = UA;
    ab.U_in = UB;
    CUtensorMap mA, mB, mX, mX2;
    if (!make_maps(aa, &mA, &mX) || !make_maps(ab, &mB, &mX2)) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(gbar, 0, 3 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    void *args[] = {&mA, &mB, &mX, &aa, &UA, &UB, &iters, &gbar};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(k_step_2d_loop<C, M2>), dim3(grid),
                                    dim3(kStepThreads), args, 0, st);
    if (e == cudaSuccess) {
        *used = true;
        return cudaSuccess;
    }
    // a refused cooperative launch (configuration, not a device fault): clear
    // the error and let the caller launch one step at a time
    (void)cudaGetLastError();
    return cudaSuccess;
}

// The iterations of one 2D state in one cooperative launch (k_step_2d_loop);
// *used = false (and nothing launched) when the CTAs cannot all be resident.
cudaError_t launch_2d_loop(const StepArgs &a0, int C, float4 *UA, float4 *UB, int iters, unsigned *gbar,
                           cudaStream_t st, bool *used) {
    *used = false;
    StepArgs a = a0;
    if (a.nz != 1 || a.v != 1 || a.hf) return cudaErrorInvalidValue;
    a.tiles_x = (a.nx + kTX - 1) / kTX;
    a.tiles_y = (a.ny + kTY - 1) / kTY;
    a.z_lo = 0; a.nz_t = 1; a.goff = 0; a.nz_g = 1;
    a.nblk = step_nblk(a.nx, a.ny, 1, true, 1);
    a.in_idx = nullptr; a.out_idx = nullptr; a.stats = nullptr; a.stop = nullptr;
    const bool m2 = a.m == 2.0f;
    switch (C) {
        case 2: return m2 ? launch_2d_loop_t<2, true>(a, UA, UB, iters, gbar, st, used)
                          : launch_2d_loop_t<2, false>(a, UA, UB, iters, gbar, st, used);
        case 3: return m2 ? launch_2d_loop_t<3, true>(a, UA, UB, iters, gbar, st, used)
                          : launch_2d_loop_t<3, false>(a, UA, UB, iters, gbar, st, used);
        case 4: return m2 ? launch_2d_loop_t<4, true>(a, UA, UB, iters, gbar, st, used)
                          : launch_2d_loop_t<4, false>(a, UA, UB, iters, gbar, st, used);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_step(const StepArgs &a0, int C, bool stencil, int P, cudaStream_t st) {
    StepArgs a = a0;
    a.tiles_x = (a.nx + kTX - 1) / kTX;
    a.tiles_y = (a.ny + kTY - 1) / kTY;
    if (a.canonical) {  // whole volume in the slab mode's canonical decomposition
        a.z_lo = 0;
        a.nz_t = a.nz;
        a.goff = 0;
        a.nz_g = a.nz;
        a.tz = slab_tz(a.nx, a.ny, a.nz);
        a.zchunks = (a.nz + a.tz - 1) / a.tz;
        a.nblk = a.tiles_x * a.tiles_y * a.zchunks;
    } else if (a.nz_g <= 0) {  // whole volume: targets are all planes
        a.z_lo = 0;
        a.nz_t = a.nz;
        a.goff = 0;
        a.nz_g = a.nz;
        a.zchunks = step_zchunks(a.nx, a.ny, a.nz, P);
        a.tz = (a.nz + a.zchunks - 1) / a.zchunks;
        a.nblk = step_nblk(a.nx, a.ny, a.nz, stencil, P);
    } else {  // z-slab: global chunks of slab_tz planes
        if (!stencil) return cudaErrorInvalidValue;
        a.tz = slab_tz(a.nx, a.ny, a.nz_g);
        a.zchunks = (a.nz_t + a.tz - 1) / a.tz;
        a.nblk = a.tiles_x * a.tiles_y * a.zchunks;
    }
    if (stencil && a.nz == 1 && a.nz_g == 1 && !a.hf && a.v == 1)  // plain 2D image: k_step_2d's blocks
        a.nblk = step_nblk(a.nx, a.ny, 1, true, P);
    if (stencil && a.v >= 2) return launch_step_shells(a, C, P, st);
    const bool m2 = (a.m == 2.0f) || a.hf != nullptr;  // the H, F pass does not depend on m
    switch (C) {
        case 2: return m2 ? launch_t<2, true>(a, stencil, P, st) : launch_t<2, false>(a, stencil, P, st);
        case 3: return m2 ? launch_t<3, true>(a, stencil, P, st) : launch_t<3, false>(a, stencil, P, st);
        case 4: return m2 ? launch_t<4, true>(a, stencil, P, st) : launch_t<4, false>(a, stencil, P, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pifcm
