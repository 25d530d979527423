// step_v2.cu -- the IFCM step with two neighbourhood shells (v = 2, NEXT-2).
//
// Eq. 9-10 (reading R2): the neighbourhood of voxel i is split
// into Chebyshev shells r = 1 (26 voxels) and r = 2 (98 voxels) of the 5x5x5
// cube; every shell is normalised on its own and weighted by Eq. 10's
//   W_r = e^{-r/h} / sum_{s=1..v} e^{-s/h}:
//   H_ij = sum_r W_r sum_{k in r} u_kj g_ik / sum_{k in r} g_ik     (Eq. 5, 6)
//   F_ij = sum_r W_r sum_{k in r} u_kj^2 q2_ik / sum_{k in r} q2_ik (Eq. 7, 8)
// (a shell whose g's are all zero contributes 0 to H, R3), then Eq. 4, Eq. 2,
// Eq. 3 / Eq. 1 exactly as the v = 1 kernel (step.cu), whose structure this
// kernel follows: a 32 x 16 voxel tile per CTA marching a z-chunk, planes
// z-2 .. z+2 of the haloed U and x tiles in a 7-stage TMA ring, 4 rows per
// thread.  Per voxel the 124 neighbours are visited explicitly (the Eq. 7
// weights are compile-time constants per offset); per-shell G is recovered
// as sum_j Hn_rj (rows of U sum to 1) and per-shell Qs is a closed form of
// the in-bounds offsets per axis.  Voxels whose memberships are sensitive to
// the fp32 factors (K > kKMax) are re-evaluated in fp64 by the
// warp from the definitions.
#include "step_common.cuh"

namespace pifcm {

constexpr int kV = 2;
constexpr int kSX2 = kTX + 2 * kV;        // 36 haloed voxels per tile row
constexpr int kSY2 = kTY + 2 * kV;        // 20 haloed rows
constexpr int kSXP2 = 40;                 // x rows from x0 - 4 (16-byte aligned TMA start)
constexpr int kXOff2 = 4;
constexpr int kU2Bytes = kSX2 * kSY2 * 16;  // 11520
constexpr int kX2Bytes = kSXP2 * kSY2 * 4;  // 3200
constexpr int kRing2 = 7;                   // planes z-2 .. z+2 in use, 2 prefetching
constexpr int kV2Smem = kRing2 * (kU2Bytes + kX2Bytes) + 128;
constexpr int kV2MinBlocks = 2;

__device__ __forceinline__ void tma4(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2,
                                     int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// In-bounds offset moments of one axis within radius R: count, sum d^2, sum d^4.
__device__ __forceinline__ void axis_moments(int X, int n, int R, float &m0, float &m2, float &m4) {
    m0 = 0.f; m2 = 0.f; m4 = 0.f;
    for (int d = -R; d <= R; ++d) {
        if (X + d < 0 || X + d >= n) continue;
        const float d2 = (float)(d * d);
        m0 += 1.f; m2 += d2; m4 += d2 * d2;
    }
}
// Sum of the Eq. 7 weights q2 (R1) over the in-bounds part of the cube of radius R.
__device__ __forceinline__ float box_q2(float x0, float x2, float x4, float y0, float y2, float y4, float z0,
                                        float z2, float z4, bool lit) {
    const float sq = x2 * y0 * z0 + x0 * y2 * z0 + x0 * y0 * z2;
    if (!lit) return sq;
    return x4 * y0 * z0 + x0 * y4 * z0 + x0 * y0 * z4 + 2.f * (x2 * y2 * z0 + x2 * y0 * z2 + x0 * y2 * z2);
}
// Eq. 7 denominators of shell 1 and shell 2 at voxel (X, Y, Z).
__device__ __forceinline__ void shell_q(int X, int Y, int Z, int nx, int ny, int nz, bool lit, float &q1,
                                        float &q2) {
    float a0, a2, a4, b0, b2, b4, c0, c2, c4;
    axis_moments(X, nx, 1, a0, a2, a4);
    axis_moments(Y, ny, 1, b0, b2, b4);
    axis_moments(Z, nz, 1, c0, c2, c4);
    q1 = box_q2(a0, a2, a4, b0, b2, b4, c0, c2, c4, lit);  // the centre has q2 = 0
    axis_moments(X, nx, 2, a0, a2, a4);
    axis_moments(Y, ny, 2, b0, b2, b4);
    axis_moments(Z, nz, 2, c0, c2, c4);
    q2 = box_q2(a0, a2, a4, b0, b2, b4, c0, c2, c4, lit) - q1;
}

// fp64 re-evaluation of the Eq. 4 factors of one voxel by the whole warp:
// lane l takes the cube offsets l, l+32, l+64, l+96 (< 125, not the centre).
template <int C>
__device__ __forceinline__ float4 attraction_coop_v2(const float4 *const (&Us)[5], const float *const (&Xs)[5],
                                                     int row, int col, int gx, int gy, int gz, int nx, int ny,
                                                     int nz, double lam, double xi, double W1, double W2,
                                                     bool lit) {
    const int lane = threadIdx.x & 31;
    double v[4 + 4 * kMaxC];
#pragma unroll
    for (int i = 0; i < 4 + 4 * kMaxC; ++i) v[i] = 0.0;
    const double xr = (double)Xs[2][row * kSXP2 + col + kXOff2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int o = lane + 32 * k;
        if (o >= 125 || o == 62) continue;
        const int dz = o / 25 - 2, dy = (o / 5) % 5 - 2, dx = o % 5 - 2;
        if (gx + dx < 0 || gx + dx >= nx || gy + dy < 0 || gy + dy >= ny || gz + dz < 0 || gz + dz >= nz) continue;
        const int ad = max(max(abs(dx), abs(dy)), abs(dz));
        const int s = ad - 1;
        // plane pointer by selection (no dynamic indexing of the pointer arrays,
        // which would put them in local memory for the whole kernel)
        const float4 *Uk = dz == -2 ? Us[0] : dz == -1 ? Us[1] : dz == 0 ? Us[2] : dz == 1 ? Us[3] : Us[4];
        const float *Xk = dz == -2 ? Xs[0] : dz == -1 ? Xs[1] : dz == 0 ? Xs[2] : dz == 1 ? Xs[3] : Xs[4];
        const float4 u = Uk[(row + dy) * kSX2 + col + 2 + dx];
        const double g = fabs(xr - (double)Xk[(row + dy) * kSXP2 + col + kXOff2 + dx]);  // Eq. 6
        const double q = (double)(dx * dx + dy * dy + dz * dz);
        const double q2 = lit ? q * q : q;                                                      // Eq. 8, R1
        const double uk[4] = {u.x, u.y, u.z, u.w};
        // compile-time indices only (a runtime shell index would move v[] to local memory)
        const double g0 = s == 0 ? g : 0.0, g1 = s == 0 ? 0.0 : g;
        const double q0 = s == 0 ? q2 : 0.0, q1 = s == 0 ? 0.0 : q2;
        v[0] += g0;
        v[1] += g1;
        v[2] += q0;
        v[3] += q1;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            v[4 + j] += uk[j] * g0;                                   // Eq. 5 numerators
            v[4 + kMaxC + j] += uk[j] * g1;
            v[4 + 2 * kMaxC + j] += uk[j] * uk[j] * q0;               // Eq. 7 numerators
            v[4 + 3 * kMaxC + j] += uk[j] * uk[j] * q1;
        }
    }
#pragma unroll
    for (int i = 0; i < 4 + 4 * kMaxC; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
    float out[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
    for (int j = 0; j < C; ++j) {
        double H = 0.0, F = 0.0;
        if (v[0] > 0.0) H = __dadd_rn(H, __dmul_rn(W1, v[4 + j] / v[0]));               // Eq. 5, R3
        if (v[1] > 0.0) H = __dadd_rn(H, __dmul_rn(W2, v[4 + kMaxC + j] / v[1]));
        if (v[2] > 0.0) F = __dadd_rn(F, __dmul_rn(W1, v[4 + 2 * kMaxC + j] / v[2]));   // Eq. 7
        if (v[3] > 0.0) F = __dadd_rn(F, __dmul_rn(W2, v[4 + 3 * kMaxC + j] / v[3]));
        const double av = __dadd_rn(__dadd_rn(1.0, -__dmul_rn(lam, H)), -__dmul_rn(xi, F));  // Eq. 4
        out[j] = (float)fmax(av, (double)kAFloor);                                          // R4
    }
    return make_float4(out[0], out[1], out[2], out[3]);
}

// HF: the ANCHORED / LEADER pass -- write the shell-weighted H and F of
// every voxel (two float4, as the v = 1 kernel's HF instance) instead of a step.
template <int C, bool M2, bool DU, bool QL, bool HF = false>
__global__ void __launch_bounds__(kStepThreads, kV2MinBlocks)
    k_step_v2(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX, const StepArgs a) {
    constexpr int NP = (C + 1) / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *base = smem_raw;
    auto sUst = [&](int s) { return reinterpret_cast<float4 *>(base + s * kU2Bytes); };
    auto sXst = [&](int s) { return reinterpret_cast<float *>(base + kRing2 * kU2Bytes + s * kX2Bytes); };
    __shared__ __align__(8) uint64_t full[kRing2];
    __shared__ int released[kRing2];

    const int p = blockIdx.z;
    if (a.stop && *a.stop) return;
    if (a.stats && a.stats[4 * p + 3] != 0.0) return;
    const int tile = blockIdx.x;
    const int x0 = (tile % a.tiles_x) * kTX;
    const int y0 = (tile / a.tiles_x) * kTY;
    const int zb = a.z_lo + blockIdx.y * a.tz;
    const int ze = min(zb + a.tz, a.z_lo + a.nz_t);
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    const int slot = a.in_idx ? a.in_idx[p] : p;

    if (tid == 0) {
        for (int s = 0; s < kRing2; ++s) {
            mbar_init(&full[s], 1);
            released[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const CUtensorMap *pmU = &tmU, *pmX = &tmX;
    const int q_first = zb - kV;
#define PIFCM_ISSUE2(q_)                                                              \
    do {                                                                              \
        const int s_ = ((q_) - q_first) % kRing2;                                     \
        mbar_expect_tx(&full[s_], kU2Bytes + kX2Bytes);                               \
        tma4(sUst(s_), pmU, &full[s_], 4 * (x0 - kV), y0 - kV, (q_), slot);           \
        tma3(sXst(s_), pmX, &full[s_], x0 - kXOff2, y0 - kV, (q_));                   \
    } while (0)
    if (tid == 0)
        for (int q = q_first; q <= min(q_first + kRing2 - 1, ze - 1 + kV); ++q) PIFCM_ISSUE2(q);

    float4 *Uout = a.U_out + (long long)(a.out_idx ? a.out_idx[p] : p) * a.nvox;
    const long long plane = (long long)a.nx * a.ny;
    float2 c2[2];
    c2[0] = make_float2(a.centers[4 * p + 0], a.centers[4 * p + 1]);
    c2[1] = make_float2(a.centers[4 * p + 2], a.centers[4 * p + 3]);
    const float lam = (float)a.lam_xi[2 * p], xi = (float)a.lam_xi[2 * p + 1];
    const float2 nlam2 = make_float2(-lam, -lam), nxi2 = make_float2(-xi, -xi);
    const int gx = x0 + tx;
    unsigned vmask = 0u;
#pragma unroll
    for (int r = 0; r < kRY; ++r)
        if (gx < a.nx && y0 + ty * kRY + r < a.ny) vmask |= 1u << r;
    float2 num2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float2 den2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float Jacc = 0.f, duacc = 0.f;
    // interior Eq. 7 denominators (closed forms; boundary voxels below)
    const float q1i = QL ? 126.f : 54.f, q2i = QL ? 5424.f : 696.f;

    for (int q = zb - kV; q < zb + kV && q < ze + kV; ++q) {  // planes zb-2 .. zb+1 (TMA completes in any order)
        const int l = q - q_first;
        mbar_wait(&full[l % kRing2], (l / kRing2) & 1);
    }
    for (int z = zb; z < ze; ++z) {
        const int lz = z - q_first;
        mbar_wait(&full[(lz + kV) % kRing2], ((lz + kV) / kRing2) & 1);
        const float4 *Up[5];
        const float *Xp[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            const int s = (lz - kV + d) % kRing2;
            Up[d] = sUst(s);
            Xp[d] = sXst(s);
        }
        float xr[kRY];
#pragma unroll
        for (int r = 0; r < kRY; ++r) xr[r] = Xp[2][(ty * kRY + kV + r) * kSXP2 + tx + kXOff2];

        float2 hn[2][kRY][NP], fn[2][kRY][NP];
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int r = 0; r < kRY; ++r)
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    hn[s][r][q] = make_float2(0.f, 0.f);
                    fn[s][r][q] = make_float2(0.f, 0.f);
                }
#pragma unroll
        for (int dz = -kV; dz <= kV; ++dz) {
            const float4 *Us = Up[dz + kV];
            const float *Xs = Xp[dz + kV];
#pragma unroll
            for (int dx = -kV; dx <= kV; ++dx) {
#pragma unroll
                for (int t = 0; t < kRY + 2 * kV; ++t) {
                    const float4 uk = Us[(ty * kRY + t) * kSX2 + tx + kV + dx];
                    const float xk = Xs[(ty * kRY + t) * kSXP2 + tx + kXOff2 + dx];
                    const float2 u01 = make_float2(uk.x, uk.y), u23 = make_float2(uk.z, uk.w);
                    const float2 s01 = __fmul2_rn(u01, u01);
                    const float2 s23 = NP > 1 ? __fmul2_rn(u23, u23) : make_float2(0.f, 0.f);
#pragma unroll
                    for (int r = 0; r < kRY; ++r) {
                        const int dy = t - kV - r;
                        if (dy < -kV || dy > kV) continue;
                        if (dx == 0 && dy == 0 && dz == 0) continue;  // Eq. 9: k != i
                        const int ad = max(max(dx < 0 ? -dx : dx, dy < 0 ? -dy : dy), dz < 0 ? -dz : dz);
                        const int s = ad - 1;                         // shell (R2)
                        const int qq = dx * dx + dy * dy + dz * dz;
                        const float w = QL ? (float)(qq * qq) : (float)qq;  // Eq. 8, R1
                        const float g = fabsf(xr[r] - xk);             // Eq. 6
                        const float2 g2 = make_float2(g, g), w2 = make_float2(w, w);
                        hn[s][r][0] = __ffma2_rn(u01, g2, hn[s][r][0]);  // Eq. 5 numerators
                        fn[s][r][0] = __ffma2_rn(s01, w2, fn[s][r][0]);  // Eq. 7 numerators
                        if (NP > 1) {
                            hn[s][r][1] = __ffma2_rn(u23, g2, hn[s][r][1]);
                            fn[s][r][1] = __ffma2_rn(s23, w2, fn[s][r][1]);
                        }
                    }
                }
            }
        }

        // ---- per-voxel epilogue
        const int gz = z + a.goff;
        const bool zin = gz >= kV && gz < a.nz_g - kV;
        float4 *Uz = Uout + (long long)z * plane + (long long)(y0 + ty * kRY) * a.nx + gx;
        unsigned band_bits = 0u;
#pragma unroll
        for (int r = 0; r < kRY; ++r) {
            const int gy = y0 + ty * kRY + r;
            float Q1 = q1i, Q2 = q2i;
            if (!(zin && gy >= kV && gy < a.ny - kV && gx >= kV && gx < a.nx - kV))
                shell_q(gx, gy, gz, a.nx, a.ny, a.nz_g, QL, Q1, Q2);
            float G1 = hn[0][r][0].x + hn[0][r][0].y, G2 = hn[1][r][0].x + hn[1][r][0].y;
            if (C > 2) { G1 += hn[0][r][NP - 1].x; G2 += hn[1][r][NP - 1].x; }
            if (C > 3) { G1 += hn[0][r][NP - 1].y; G2 += hn[1][r][NP - 1].y; }  // = sum_k g (rows sum to 1)
            const float h1 = G1 > 0.f ? a.w1 * rcp_approx(G1) : 0.f, h2 = G2 > 0.f ? a.w2 * rcp_approx(G2) : 0.f;
            const float f1 = Q1 > 0.f ? a.w1 / Q1 : 0.f, f2 = Q2 > 0.f ? a.w2 / Q2 : 0.f;
            float2 A[2], Ar[2];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const float2 H = __ffma2_rn(hn[1][r][q], make_float2(h2, h2),
                                            __fmul2_rn(hn[0][r][q], make_float2(h1, h1)));  // Eq. 5, Eq. 10
                const float2 F = __ffma2_rn(fn[1][r][q], make_float2(f2, f2),
                                            __fmul2_rn(fn[0][r][q], make_float2(f1, f1)));  // Eq. 7, Eq. 10
                Ar[q] = __ffma2_rn(H, nlam2, __ffma2_rn(F, nxi2, make_float2(1.f, 1.f)));  // Eq. 4
                A[q].x = fmaxf(Ar[q].x, kAFloor);                                           // R4
                A[q].y = fmaxf(Ar[q].y, kAFloor);
            }
            if (NP == 1) { A[1] = make_float2(1.f, 1.f); Ar[1] = A[1]; }
            if (HF) {  // particle-invariant H, F of this state (Eq. 5, 7, 10)
                if ((vmask >> r) & 1u) {
                    float2 Hh[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                    float2 Ff[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        Hh[q] = __ffma2_rn(hn[1][r][q], make_float2(h2, h2), __fmul2_rn(hn[0][r][q], make_float2(h1, h1)));
                        Ff[q] = __ffma2_rn(fn[1][r][q], make_float2(f2, f2), __fmul2_rn(fn[0][r][q], make_float2(f1, f1)));
                    }
                    float4 *o = a.hf + 2 * ((long long)z * plane + (long long)gy * a.nx + gx);
                    o[0] = make_float4(Hh[0].x, Hh[0].y, Hh[1].x, Hh[1].y);
                    o[1] = make_float4(Ff[0].x, Ff[0].y, Ff[1].x, Ff[1].y);
                }
                continue;
            }
            const Memb mb = memb_compute<C, M2>(xr[r], c2, A, a.m, a.inv_m1, Ar);
            const bool valid = (vmask >> r) & 1u;
            const bool band = valid && !(mb.K <= kKMax);
            band_bits |= band ? (1u << r) : 0u;
            if (valid && !band) {
                memb_accumulate<C, M2>(mb, xr[r], a.m, num2, den2, Jacc);
                const float4 un = make_float4(mb.u[0], mb.u[1], mb.u[2], mb.u[3]);
                if (DU) {
                    const float4 uo = Up[2][(ty * kRY + kV + r) * kSX2 + tx + kV];
                    duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                               fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                }
                Uz[(long long)r * a.nx] = un;
            }
        }
        unsigned lanes = __ballot_sync(0xffffffffu, band_bits != 0u);
        while (lanes) {
            const int L = __ffs(lanes) - 1;
            lanes &= lanes - 1;
            unsigned bits = __shfl_sync(0xffffffffu, band_bits, L);
            while (bits) {
                const int r = __ffs(bits) - 1;
                bits &= bits - 1;
                const int row = ty * kRY + kV + r;
                const int gxL = x0 + L, gy = y0 + ty * kRY + r;
                const float4 a4 = attraction_coop_v2<C>(Up, Xp, row, L, gxL, gy, gz, a.nx, a.ny, a.nz_g,
                                                        a.lam_xi[2 * p], a.lam_xi[2 * p + 1], a.w1d, a.w2d, QL);
                if (tx == L) {
                    const float2 A[2] = {make_float2(a4.x, a4.y), make_float2(a4.z, a4.w)};
                    const float xv = Xp[2][row * kSXP2 + L + kXOff2];
                    const float4 un = membership2<C, M2>(xv, c2, A, a.m, a.inv_m1, num2, den2, Jacc);
                    if (DU) {
                        const float4 uo = Up[2][row * kSX2 + L + kV];
                        duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                                   fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                    }
                    Uout[(long long)z * plane + (long long)gy * a.nx + gxL] = un;
                }
            }
        }
        // release plane z-2; the last warp refills its stage with plane z-2+kRing2
        __syncwarp();
        if (tx == 0) {
            const int sm = (lz - kV) % kRing2;
            const int old = atomicAdd(&released[sm], 1);
            if (old == kWarpsY - 1) {
                released[sm] = 0;
                if (z - kV + kRing2 <= ze - 1 + kV) PIFCM_ISSUE2(z - kV + kRing2);
            }
        }
    }
#undef PIFCM_ISSUE2
    if (HF) return;  // no reductions: H, F only
    float num[kMaxC] = {num2[0].x, num2[0].y, num2[1].x, num2[1].y};
    float den[kMaxC] = {den2[0].x, den2[0].y, den2[1].x, den2[1].y};
    const int blk = blockIdx.x + gridDim.x * blockIdx.y;
    block_partials<kWarpsY>(num, den, Jacc, duacc, a.partials + ((long long)p * a.nblk + blk) * kNR);
    finalize_if_last<kStepThreads>(a, p, a.nblk);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn2() {
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

static bool make_maps2(const StepArgs &a, CUtensorMap *mU, CUtensorMap *mX) {
    auto enc = encode_fn2();
    if (!enc) return false;
    const cuuint64_t du[4] = {4ull * a.nx, (cuuint64_t)a.ny, (cuuint64_t)a.nz, (cuuint64_t)a.n_in_states};
    const cuuint64_t su[3] = {16ull * a.nx, 16ull * a.nx * a.ny, 16ull * (cuuint64_t)a.nvox};
    const cuuint32_t bu[4] = {4 * kSX2, kSY2, 1, 1};
    const cuuint32_t e5[5] = {1, 1, 1, 1, 1};
    if (enc(mU, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float4 *>(a.U_in), du, su, bu, e5,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const cuuint64_t dx[3] = {(cuuint64_t)a.nx, (cuuint64_t)a.ny, (cuuint64_t)a.nz};
    const cuuint64_t sx[2] = {4ull * a.pitch, 4ull * a.pitch * a.ny};
    const cuuint32_t bx[3] = {kSXP2, kSY2, 1};
    return enc(mX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(a.x), dx, sx, bx, e5,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C, bool M2, bool DU, bool QL, bool HF = false>
static cudaError_t launch_v2_t(const StepArgs &a, int P, cudaStream_t st) {
    // the dynamic shared-memory opt-in is per device: remember it per device
    static unsigned long long attr_set = 0ull;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    if (dev < 64 && !(attr_set & (1ull << dev))) {
        const cudaError_t e = cudaFuncSetAttribute(k_step_v2<C, M2, DU, QL, HF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   kV2Smem);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << dev;
    }
    CUtensorMap mU, mX;
    if (!make_maps2(a, &mU, &mX)) return cudaErrorInvalidValue;
    dim3 grid(a.tiles_x * a.tiles_y, a.zchunks, P);
    k_step_v2<C, M2, DU, QL, HF><<<grid, kStepThreads, kV2Smem, st>>>(mU, mX, a);
    return cudaGetLastError();
}

template <int C, bool M2>
static cudaError_t launch_v2_c(const StepArgs &a, int P, cudaStream_t st) {
    const bool ql = a.q_mode == 0;
    if (a.hf) return ql ? launch_v2_t<C, true, false, true, true>(a, P, st)
                        : launch_v2_t<C, true, false, false, true>(a, P, st);
    if (a.want_du) return ql ? launch_v2_t<C, M2, true, true>(a, P, st) : launch_v2_t<C, M2, true, false>(a, P, st);
    return ql ? launch_v2_t<C, M2, false, true>(a, P, st) : launch_v2_t<C, M2, false, false>(a, P, st);
}

// The decomposition fields of `a` (tiles, z-chunks, nblk) are set by launch_step.
cudaError_t launch_step_v2(const StepArgs &a, int C, int P, cudaStream_t st) {
    const bool m2 = (a.m == 2.0f) || a.hf != nullptr;  // the H, F pass does not depend on m
    switch (C) {
        case 2: return m2 ? launch_v2_c<2, true>(a, P, st) : launch_v2_c<2, false>(a, P, st);
        case 3: return m2 ? launch_v2_c<3, true>(a, P, st) : launch_v2_c<3, false>(a, P, st);
        case 4: return m2 ? launch_v2_c<4, true>(a, P, st) : launch_v2_c<4, false>(a, P, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pifcm
