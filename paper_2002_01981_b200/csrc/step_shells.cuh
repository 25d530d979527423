// step_shells.cuh -- the IFCM step with v = 2 or 3 neighbourhood shells (NEXT-2).
// Instantiated per (v, C) in step_shells_v<V>_c<C>.cu (one translation unit
// each, so the parallel build compiles them side by side); dispatched by
// launch_step_shells (step_shells.cu).
//
// Eq. 9-10 (reading R2): the neighbourhood of voxel i is split
// into Chebyshev shells r = 1 (26 voxels), r = 2 (98), r = 3 (218) of the
// (2v+1)^3 cube; every shell is normalised on its own and weighted by Eq. 10's
//   W_r = e^{-r/h} / sum_{s=1..v} e^{-s/h}:
//   H_ij = sum_r W_r sum_{k in r} u_kj g_ik / sum_{k in r} g_ik     (Eq. 5, 6)
//   F_ij = sum_r W_r sum_{k in r} u_kj^2 q2_ik / sum_{k in r} q2_ik (Eq. 7, 8)
// (a shell whose g's are all zero contributes 0 to H, R3), then Eq. 4, Eq. 2,
// Eq. 3 / Eq. 1 exactly as the v = 1 kernel (step.cu), whose structure this
// kernel follows: a 32 x 16 voxel tile per CTA marching a z-chunk, planes
// z-v .. z+v of the haloed U and x tiles in a (2v+3)-stage TMA ring, 4 rows
// per thread.  Per voxel the 124 (342) neighbours are visited explicitly (the
// Eq. 7 weights are compile-time constants per offset); per-shell G is
// recovered as sum_j Hn_rj (rows of U sum to 1) and per-shell Qs is a closed
// form of the in-bounds offsets per axis.  Voxels whose memberships are sensitive to
// the fp32 factors (K > kKMax) are re-evaluated in fp64 by the
// warp from the definitions.
#pragma once
#include "step_common.cuh"

namespace pifcm {

// geometry of the v-shell kernel
template <int V>
struct Shells {
    static constexpr int SX = kTX + 2 * V;       // haloed voxels per tile row
    static constexpr int SY = kTY + 2 * V;       // haloed rows
    static constexpr int SXP = 40;               // x rows from x0 - 4 (16-byte aligned TMA start), >= 32 + 4 + V
    static constexpr int XOFF = 4;
    static constexpr int UBYTES = SX * SY * 16;  // TMA box bytes: 11520 (v = 2), 13376 (v = 3)
    static constexpr int XBYTES = SXP * SY * 4;
    static constexpr int UPAD = (UBYTES + 127) / 128 * 128;  // stage strides: TMA destinations 128-byte aligned
    static constexpr int XPAD = (XBYTES + 127) / 128 * 128;
    static constexpr int RING = 2 * V + 3;       // planes z-v .. z+v in use, 2 prefetching
    static constexpr int SMEM = RING * (UPAD + XPAD) + 128;
    static constexpr int MINBLOCKS = V == 2 ? 2 : 1;
    static constexpr int CUBE = (2 * V + 1) * (2 * V + 1) * (2 * V + 1);
};
static_assert(Shells<3>::SXP >= kTX + 4 + 3, "x box too narrow");

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
// Eq. 7 denominators of shells 1 .. V at voxel (X, Y, Z): the in-bounds
// q2 sums of the cubes of radius r, differenced.
template <int V>
__device__ __forceinline__ void shell_q(int X, int Y, int Z, int nx, int ny, int nz, bool lit, float (&q)[V]) {
    float prev = 0.f;  // the centre has q2 = 0
#pragma unroll
    for (int r = 1; r <= V; ++r) {
        float a0, a2, a4, b0, b2, b4, c0, c2, c4;
        axis_moments(X, nx, r, a0, a2, a4);
        axis_moments(Y, ny, r, b0, b2, b4);
        axis_moments(Z, nz, r, c0, c2, c4);
        const float box = box_q2(a0, a2, a4, b0, b2, b4, c0, c2, c4, lit);
        q[r - 1] = box - prev;
        prev = box;
    }
}

// fp64 re-evaluation of the Eq. 4 factors of one voxel by the whole warp:
// lane l takes the cube offsets l, l+32, ... (< (2V+1)^3, not the centre).
// Us / Xs: the 2V+1 planes z-V .. z+V.
template <int C, int V>
__device__ __forceinline__ float4 attraction_coop_shells(const float4 *const (&Us)[2 * V + 1],
                                                         const float *const (&Xs)[2 * V + 1], int row, int col,
                                                         int gx, int gy, int gz, int nx, int ny, int nz, double lam,
                                                         double xi, const double *W, bool lit) {
    using S = Shells<V>;
    constexpr int NV = 2 * V + 2 * V * kMaxC;  // per shell: sum g, sum q2, then the numerators
    const int lane = threadIdx.x & 31;
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = 0.0;
    const double xr = (double)Xs[V][row * S::SXP + col + S::XOFF];
    constexpr int W2 = 2 * V + 1;
#pragma unroll
    for (int k = 0; k < (S::CUBE + 31) / 32; ++k) {
        const int o = lane + 32 * k;
        if (o >= S::CUBE || o == S::CUBE / 2) continue;
        const int dz = o / (W2 * W2) - V, dy = (o / W2) % W2 - V, dx = o % W2 - V;
        if (gx + dx < 0 || gx + dx >= nx || gy + dy < 0 || gy + dy >= ny || gz + dz < 0 || gz + dz >= nz) continue;
        const int ad = max(max(abs(dx), abs(dy)), abs(dz));
        // plane pointer by selection (no dynamic indexing of the pointer arrays,
        // which would put them in local memory for the whole kernel)
        const float4 *Uk = Us[0];
        const float *Xk = Xs[0];
#pragma unroll
        for (int d = 1; d <= 2 * V; ++d)
            if (dz + V == d) { Uk = Us[d]; Xk = Xs[d]; }
        const float4 u = Uk[(row + dy) * S::SX + col + V + dx];
        const double g = fabs(xr - (double)Xk[(row + dy) * S::SXP + col + S::XOFF + dx]);  // Eq. 6
        const double q = (double)(dx * dx + dy * dy + dz * dz);
        const double q2 = lit ? q * q : q;                                                      // Eq. 8, R1
        const double uk[4] = {u.x, u.y, u.z, u.w};
        // compile-time indices only (a runtime shell index would move v[] to local memory)
#pragma unroll
        for (int s = 0; s < V; ++s) {
            const double gs = ad == s + 1 ? g : 0.0, qs = ad == s + 1 ? q2 : 0.0;
            v[s] += gs;
            v[V + s] += qs;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                v[2 * V + s * kMaxC + j] += uk[j] * gs;                       // Eq. 5 numerators
                v[2 * V + V * kMaxC + s * kMaxC + j] += uk[j] * uk[j] * qs;   // Eq. 7 numerators
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
    float out[4] = {1.f, 1.f, 1.f, 1.f};
#pragma unroll
    for (int j = 0; j < C; ++j) {
        double H = 0.0, F = 0.0;
#pragma unroll
        for (int s = 0; s < V; ++s) {
            if (v[s] > 0.0) H = __dadd_rn(H, __dmul_rn(W[s], v[2 * V + s * kMaxC + j] / v[s]));                 // Eq. 5, R3
            if (v[V + s] > 0.0) F = __dadd_rn(F, __dmul_rn(W[s], v[2 * V + V * kMaxC + s * kMaxC + j] / v[V + s]));  // Eq. 7
        }
        const double av = __dadd_rn(__dadd_rn(1.0, -__dmul_rn(lam, H)), -__dmul_rn(xi, F));  // Eq. 4
        out[j] = (float)fmax(av, (double)kAFloor);                                          // R4
    }
    return make_float4(out[0], out[1], out[2], out[3]);
}

// HF: the ANCHORED / LEADER pass -- write the shell-weighted H and F of
// every voxel (two float4, as the v = 1 kernel's HF instance) instead of a step.
template <int C, bool M2, bool DU, bool QL, int V, bool HF = false>
__global__ void __launch_bounds__(kStepThreads, Shells<V>::MINBLOCKS)
    k_step_shells(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX,
                  const StepArgs a) {
    using S = Shells<V>;
    constexpr int NP = (C + 1) / 2;
    constexpr int RING = S::RING;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *base = smem_raw;
    auto sUst = [&](int s) { return reinterpret_cast<float4 *>(base + s * S::UPAD); };
    auto sXst = [&](int s) { return reinterpret_cast<float *>(base + RING * S::UPAD + s * S::XPAD); };
    __shared__ __align__(8) uint64_t full[RING];
    __shared__ int released[RING];

    // grid (tile, state, chunk) as the v = 1 kernel: the states of a
    // tile-chunk share its intensity planes in L2
    const int p = blockIdx.y, chunk = blockIdx.z;
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
        for (int s = 0; s < RING; ++s) {
            mbar_init(&full[s], 1);
            released[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const CUtensorMap *pmU = &tmU, *pmX = &tmX;
    const int q_first = zb - V;
#define PIFCM_ISSUE2(q_)                                                              \
    do {                                                                              \
        const int s_ = ((q_) - q_first) % RING;                                       \
        mbar_expect_tx(&full[s_], S::UBYTES + S::XBYTES);                             \
        tma4(sUst(s_), pmU, &full[s_], 4 * (x0 - V), y0 - V, (q_), slot);             \
        tma3(sXst(s_), pmX, &full[s_], x0 - S::XOFF, y0 - V, (q_));                   \
    } while (0)
    if (tid == 0)
        for (int q = q_first; q <= min(q_first + RING - 1, ze - 1 + V); ++q) PIFCM_ISSUE2(q);

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
    // interior Eq. 7 denominators (the closed form at a voxel far from every
    // face; boundary voxels below)
    float qint[V];
    shell_q<V>(V, V, V, 2 * V + 1, 2 * V + 1, 2 * V + 1, QL, qint);

    for (int q = zb - V; q < zb + V && q < ze + V; ++q) {  // planes zb-V .. zb+V-1 (TMA completes in any order)
        const int l = q - q_first;
        mbar_wait(&full[l % RING], (l / RING) & 1);
    }
    for (int z = zb; z < ze; ++z) {
        const int lz = z - q_first;
        mbar_wait(&full[(lz + V) % RING], ((lz + V) / RING) & 1);
        const float4 *Up[2 * V + 1];
        const float *Xp[2 * V + 1];
#pragma unroll
        for (int d = 0; d < 2 * V + 1; ++d) {
            const int s = (lz - V + d) % RING;
            Up[d] = sUst(s);
            Xp[d] = sXst(s);
        }
        float xr[kRY];
#pragma unroll
        for (int r = 0; r < kRY; ++r) xr[r] = Xp[V][(ty * kRY + V + r) * S::SXP + tx + S::XOFF];

        float2 hn[V][kRY][NP], fn[V][kRY][NP];
#pragma unroll
        for (int s = 0; s < V; ++s)
#pragma unroll
            for (int r = 0; r < kRY; ++r)
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    hn[s][r][q] = make_float2(0.f, 0.f);
                    fn[s][r][q] = make_float2(0.f, 0.f);
                }
#pragma unroll
        for (int dz = -V; dz <= V; ++dz) {
            const float4 *Us = Up[dz + V];
            const float *Xs = Xp[dz + V];
#pragma unroll
            for (int dx = -V; dx <= V; ++dx) {
#pragma unroll
                for (int t = 0; t < kRY + 2 * V; ++t) {
                    const float4 uk = Us[(ty * kRY + t) * S::SX + tx + V + dx];
                    const float xk = Xs[(ty * kRY + t) * S::SXP + tx + S::XOFF + dx];
                    const float2 u01 = make_float2(uk.x, uk.y), u23 = make_float2(uk.z, uk.w);
                    const float2 s01 = __fmul2_rn(u01, u01);
                    const float2 s23 = NP > 1 ? __fmul2_rn(u23, u23) : make_float2(0.f, 0.f);
#pragma unroll
                    for (int r = 0; r < kRY; ++r) {
                        const int dy = t - V - r;
                        if (dy < -V || dy > V) continue;
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
        const bool zin = gz >= V && gz < a.nz_g - V;
        float4 *Uz = Uout + (long long)z * plane + (long long)(y0 + ty * kRY) * a.nx + gx;
        unsigned band_bits = 0u;
#pragma unroll
        for (int r = 0; r < kRY; ++r) {
            const int gy = y0 + ty * kRY + r;
            float Qs[V];
#pragma unroll
            for (int s = 0; s < V; ++s) Qs[s] = qint[s];
            if (!(zin && gy >= V && gy < a.ny - V && gx >= V && gx < a.nx - V))
                shell_q<V>(gx, gy, gz, a.nx, a.ny, a.nz_g, QL, Qs);
            float2 H[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float2 F[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int s = 0; s < V; ++s) {
                float G = hn[s][r][0].x + hn[s][r][0].y;
                if (C > 2) G += hn[s][r][NP - 1].x;
                if (C > 3) G += hn[s][r][NP - 1].y;  // = sum_k g over shell s (rows sum to 1)
                const float hs = G > 0.f ? a.wsh[s] * rcp_approx(G) : 0.f;   // Eq. 5, Eq. 10, R3
                const float fs = Qs[s] > 0.f ? a.wsh[s] / Qs[s] : 0.f;       // Eq. 7, Eq. 10
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    H[q] = __ffma2_rn(hn[s][r][q], make_float2(hs, hs), H[q]);
                    F[q] = __ffma2_rn(fn[s][r][q], make_float2(fs, fs), F[q]);
                }
            }
            float2 A[2], Ar[2];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                Ar[q] = __ffma2_rn(H[q], nlam2, __ffma2_rn(F[q], nxi2, make_float2(1.f, 1.f)));  // Eq. 4
                A[q].x = fmaxf(Ar[q].x, kAFloor);                                                // R4
                A[q].y = fmaxf(Ar[q].y, kAFloor);
            }
            if (NP == 1) { A[1] = make_float2(1.f, 1.f); Ar[1] = A[1]; }
            if (HF) {  // particle-invariant H, F of this state (Eq. 5, 7, 10)
                if ((vmask >> r) & 1u) {
                    float4 *o = a.hf + 2 * ((long long)z * plane + (long long)gy * a.nx + gx);
                    o[0] = make_float4(H[0].x, H[0].y, NP > 1 ? H[1].x : 0.f, NP > 1 ? H[1].y : 0.f);
                    o[1] = make_float4(F[0].x, F[0].y, NP > 1 ? F[1].x : 0.f, NP > 1 ? F[1].y : 0.f);
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
                    const float4 uo = Up[V][(ty * kRY + V + r) * S::SX + tx + V];
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
                const int row = ty * kRY + V + r;
                const int gxL = x0 + L, gy = y0 + ty * kRY + r;
                const float4 a4 = attraction_coop_shells<C, V>(Up, Xp, row, L, gxL, gy, gz, a.nx, a.ny, a.nz_g,
                                                               a.lam_xi[2 * p], a.lam_xi[2 * p + 1], a.wshd, QL);
                if (tx == L) {
                    const float2 A[2] = {make_float2(a4.x, a4.y), make_float2(a4.z, a4.w)};
                    const float xv = Xp[V][row * S::SXP + L + S::XOFF];
                    const float4 un = membership2<C, M2>(xv, c2, A, a.m, a.inv_m1, num2, den2, Jacc);
                    if (DU) {
                        const float4 uo = Up[V][row * S::SX + L + V];
                        duacc = fmaxf(duacc, fmaxf(fmaxf(fabsf(un.x - uo.x), fabsf(un.y - uo.y)),
                                                   fmaxf(fabsf(un.z - uo.z), fabsf(un.w - uo.w))));
                    }
                    Uout[(long long)z * plane + (long long)gy * a.nx + gxL] = un;
                }
            }
        }
        // release plane z-V; the last warp refills its stage with plane z-V+RING
        __syncwarp();
        if (tx == 0) {
            const int sm = (lz - V) % RING;
            const int old = atomicAdd(&released[sm], 1);
            if (old == kWarpsY - 1) {
                released[sm] = 0;
                if (z - V + RING <= ze - 1 + V) PIFCM_ISSUE2(z - V + RING);
            }
        }
    }
#undef PIFCM_ISSUE2
    if (HF) return;  // no reductions: H, F only
    float num[kMaxC] = {num2[0].x, num2[0].y, num2[1].x, num2[1].y};
    float den[kMaxC] = {den2[0].x, den2[0].y, den2[1].x, den2[1].y};
    const int blk = blockIdx.x + gridDim.x * chunk;
    block_partials<kWarpsY>(num, den, Jacc, duacc, a.partials + ((long long)p * a.nblk + blk) * kNR);
    finalize_if_last<kStepThreads>(a, p, a.nblk, reinterpret_cast<double(*)[kNR]>(smem_raw));
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

template <int V>
static bool make_maps2(const StepArgs &a, CUtensorMap *mU, CUtensorMap *mX) {
    using S = Shells<V>;
    auto enc = encode_fn2();
    if (!enc) return false;
    const cuuint64_t du[4] = {4ull * a.nx, (cuuint64_t)a.ny, (cuuint64_t)a.nz, (cuuint64_t)a.n_in_states};
    const cuuint64_t su[3] = {16ull * a.nx, 16ull * a.nx * a.ny, 16ull * (cuuint64_t)a.nvox};
    const cuuint32_t bu[4] = {4 * S::SX, S::SY, 1, 1};
    const cuuint32_t e5[5] = {1, 1, 1, 1, 1};
    if (enc(mU, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float4 *>(a.U_in), du, su, bu, e5,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const cuuint64_t dx[3] = {(cuuint64_t)a.nx, (cuuint64_t)a.ny, (cuuint64_t)a.nz};
    const cuuint64_t sx[2] = {4ull * a.pitch, 4ull * a.pitch * a.ny};
    const cuuint32_t bx[3] = {S::SXP, S::SY, 1};
    return enc(mX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(a.x), dx, sx, bx, e5,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C, bool M2, bool DU, bool QL, int V, bool HF = false>
static cudaError_t launch_shells_t(const StepArgs &a, int P, cudaStream_t st) {
    // the dynamic shared-memory opt-in is per device: remember it per device
    static unsigned long long attr_set = 0ull;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    if (dev < 64 && !(attr_set & (1ull << dev))) {
        const cudaError_t e = cudaFuncSetAttribute(k_step_shells<C, M2, DU, QL, V, HF>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, Shells<V>::SMEM);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << dev;
    }
    CUtensorMap mU, mX;
    if (!make_maps2<V>(a, &mU, &mX)) return cudaErrorInvalidValue;
    dim3 grid(a.tiles_x * a.tiles_y, P, a.zchunks);
    k_step_shells<C, M2, DU, QL, V, HF><<<grid, kStepThreads, Shells<V>::SMEM, st>>>(mU, mX, a);
    return cudaGetLastError();
}

template <int C, bool M2, int V>
static cudaError_t launch_shells_c(const StepArgs &a, int P, cudaStream_t st) {
    const bool ql = a.q_mode == 0;
    if (a.hf) return ql ? launch_shells_t<C, true, false, true, V, true>(a, P, st)
                        : launch_shells_t<C, true, false, false, V, true>(a, P, st);
    if (a.want_du)
        return ql ? launch_shells_t<C, M2, true, true, V>(a, P, st) : launch_shells_t<C, M2, true, false, V>(a, P, st);
    return ql ? launch_shells_t<C, M2, false, true, V>(a, P, st) : launch_shells_t<C, M2, false, false, V>(a, P, st);
}

// One (v, C) instance family: m = 2 or general m, with / without max|du|,
// LITERAL / SQEUCLID q (R1), and the H, F pass of the fitness modes.
#define PIFCM_SHELLS_INSTANCE(V_, C_)                                                           \
    cudaError_t launch_shells_##V_##_##C_(const StepArgs &a, int P, cudaStream_t st) {          \
        const bool m2 = (a.m == 2.0f) || a.hf != nullptr; /* the H, F pass does not depend on m */ \
        return m2 ? launch_shells_c<C_, true, V_>(a, P, st) : launch_shells_c<C_, false, V_>(a, P, st); \
    }

}  // namespace pifcm
