// step_common.cuh -- device helpers shared by the stencil step kernels
// (step.cu: 26-neighbourhood, v = 1; step_v2.cu: two Chebyshev shells, v = 2):
// the per-voxel membership epilogue (Eq. 4, Eq. 2, Eq. 1 / Eq. 3 partial
// sums), the fixed-order block reduction and fused finalisation (Eq. 3 /
// Eq. 1), and the TMA / mbarrier PTX wrappers.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "pifcm_internal.cuh"

#ifndef PIFCM_KGATE
#define PIFCM_KGATE 1
#endif
#ifndef PIFCM_KGATE_UNIFORM
#define PIFCM_KGATE_UNIFORM 1
#endif

namespace pifcm {
__device__ __forceinline__ float rcp_approx(float v) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
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
        __threadfence();  // the record is visible device-wide before this CTA is counted
    }
}

// Fixed-order fp64 sum of the nblk partial records of state p, then Eq. 3
// (PAPER:57): c_j = sum u^m x / sum u^m (c_j kept if the sum < 1e-12, R9) and
// Eq. 1: J = sum of the per-voxel costs.  All NT threads of the CTA
// take part; red is NT x kNR doubles of shared memory.  The summation order
// depends on nblk and NT only, not on which CTA runs it (k_slab_finalize uses
// the same order for records gathered across z-slab ranks).
template <int NT>
__device__ __forceinline__ void finalize_state(const StepArgs &a, int p, int nblk, double (*red)[kNR]) {
    const double *src = a.partials + (long long)p * nblk * kNR;
    double v[kNR];
#pragma unroll
    for (int r = 0; r < kNR; ++r) v[r] = 0.0;
    for (int b = threadIdx.x; b < nblk; b += NT) {
#pragma unroll
        for (int r = 0; r < kNR - 1; ++r) v[r] += __ldcg(src + (long long)b * kNR + r);
        v[kNR - 1] = fmax(v[kNR - 1], __ldcg(src + (long long)b * kNR + kNR - 1));
    }
#pragma unroll
    for (int r = 0; r < kNR; ++r) red[threadIdx.x][r] = v[r];
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
#pragma unroll
            for (int r = 0; r < kNR - 1; ++r) red[threadIdx.x][r] += red[threadIdx.x + s][r];
            red[threadIdx.x][kNR - 1] = fmax(red[threadIdx.x][kNR - 1], red[threadIdx.x + s][kNR - 1]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double J = red[0][2 * kMaxC], du = red[0][2 * kMaxC + 1];
        for (int j = 0; j < a.C; ++j) {
            const double num = red[0][j], den = red[0][kMaxC + j];
            if (den >= kDenEps) a.centers[4 * p + j] = (float)(num / den);
        }
        if (a.fitness) a.fitness[p] = J;
        if (a.stats_out) {
            a.stats_out[4 * p + 0] = J;
            a.stats_out[4 * p + 1] = du;
            a.stats_out[4 * p + 2] += 1.0;
            a.stats_out[4 * p + 3] = (a.eps > 0.f && du < (double)a.eps) ? 1.0 : 0.0;
        }
        if (!isfinite(J) && a.status) atomicExch(a.status, (int)PIFCM_ENUMERIC);
        a.counters[p] = 0u;  // ready for the next launch
    }
    __syncthreads();  // red is reused by the caller
}

// Finalisation by the last CTA of state p (threadFenceReduction pattern);
// red: NT x kNR doubles of shared memory the caller no longer needs.
template <int NT>
__device__ __forceinline__ void finalize_if_last(const StepArgs &a, int p, int nblk, double (*red)[kNR]) {
    __shared__ int is_last;
    if (a.counters == nullptr) return;  // z-slab mode: records are combined across ranks
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(&a.counters[p], 1u) == (unsigned)(nblk - 1));
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    finalize_state<NT>(a, p, nblk, red);
}
template <int NT>
__device__ __forceinline__ void finalize_if_last(const StepArgs &a, int p, int nblk) {
    __shared__ double red[NT][kNR];
    finalize_if_last<NT>(a, p, nblk, red);
}

// ----------------------------------------------------------------------------
// TMA / mbarrier helpers (sm_90+ PTX, compiled for sm_100a).
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// ----------------------------------------------------------------------------
// Packed (FFMA2) epilogue of one voxel: Eq. 4 distances from the attraction
// factors A (already floored), Eq. 2 memberships, Eq. 1 / Eq. 3 partial sums.
// Cluster pairs (0,1), (2,3); for odd C the padded component is masked.
// Memberships of one voxel (Eq. 4 distances from the floored attraction
// factors A, Eq. 2), its Eq. 1 cost and its sensitivity to the factors:
//   K = sum_j |d u / d ln a_j| = sum_j u_j (1 - u_j) / ((m - 1) a_j)
// (1/a_j = w_j (x - c_j)^2 for m = 2, with w_j = d2_ij^{-1/(m-1)}); the fp32
// factors carry an absolute error <= kAErr, so K * kAErr bounds the error
// of u, and voxels with K > kKMax are re-evaluated in fp64.
struct Memb {
    float u[4];
    float Ji, K;
};
template <int C, bool M2>
__device__ __forceinline__ Memb memb_compute(float xv, const float2 (&c2)[2], const float2 (&A)[2], float m,
                                             float inv_m1, const float2 (&Ar)[2]) {
    constexpr int NP = (C + 1) / 2;
    const float2 x2 = make_float2(xv, xv);
    float d2[4], dd[4];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const float2 d = __fadd2_rn(x2, make_float2(-c2[q].x, -c2[q].y));
        const float2 s2 = __fmul2_rn(d, d);
        const float2 e = __fmul2_rn(s2, A[q]);  // Eq. 4
        d2[2 * q] = e.x;
        d2[2 * q + 1] = e.y;
        dd[2 * q] = s2.x;
        dd[2 * q + 1] = s2.y;
    }
    float w[4] = {0.f, 0.f, 0.f, 0.f}, S = 0.0f;
#pragma unroll
    for (int j = 0; j < C; ++j) {
        w[j] = M2 ? rcp_approx(d2[j]) : exp2f(-log2f(d2[j]) * inv_m1);  // d2 = 0 -> +inf
        S += w[j];
    }
    const float invS = rcp_approx(S);
    Memb r;
    float Kp[2] = {0.f, 0.f};
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const float2 wq = make_float2(w[2 * q], w[2 * q + 1]);
        const float2 uu = __fmul2_rn(wq, make_float2(invS, invS));  // Eq. 2
        r.u[2 * q] = uu.x;
        r.u[2 * q + 1] = uu.y;
    }
#if PIFCM_KGATE
    // K <= sum_j u_j (1 - u_j) / min_j |a_j| <= (1 - 1/C) / min_j |a_j|
    // (times 1/(m-1)): when that bound is below kKMax the voxel is not in the
    // band and K need not be formed (NaN factors fall through to K)
    float amin = fminf(fabsf(Ar[0].x), fabsf(Ar[0].y));
    if (NP > 1) amin = fminf(amin, fminf(fabsf(Ar[NP - 1].x), fabsf(Ar[NP - 1].y)));
#if PIFCM_KGATE_UNIFORM
    // warp-uniform decision (no reconvergence point): K is exact where formed
    const bool kneed = __any_sync(__activemask(), !(amin * kKMax >= 0.75f * (M2 ? 1.0f : inv_m1)));
#else
    const bool kneed = !(amin * kKMax >= 0.75f * (M2 ? 1.0f : inv_m1));
#endif
#else
    const bool kneed = true;
#endif
    if (kneed) {
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const float2 uu = make_float2(r.u[2 * q], r.u[2 * q + 1]);
            // u (1 - u) / |a| with the unfloored factor: a clamped factor (a << 0)
            // contributes little (its u is ~0 or ~1), an uncertain clamp (|a| ~ 0)
            // makes K huge, an unclamped small factor is weighed by 1/a
            const float2 ia = make_float2(rcp_approx(fabsf(Ar[q].x)), rcp_approx(fabsf(Ar[q].y)));
            const float2 t = __fmul2_rn(__fmul2_rn(uu, __fadd2_rn(make_float2(1.f, 1.f), make_float2(-uu.x, -uu.y))), ia);
            Kp[q] = t.x + ((2 * q + 1 < C) ? t.y : 0.f);
        }
    }
    if (NP == 1) { r.u[2] = 0.f; r.u[3] = 0.f; }
    r.K = M2 ? Kp[0] + Kp[1] : (Kp[0] + Kp[1]) * inv_m1;
    (void)dd;
    r.Ji = M2 ? invS : exp2f((1.0f - m) * log2f(S));  // Eq. 1 per voxel: S^{1-m}
    if (!(S < INFINITY)) {  // R5: a zero distance -> crisp row at the lowest such j (rare)
        int jz = C - 1;
#pragma unroll
        for (int j = C - 1; j >= 0; --j)
            if (d2[j] == 0.0f) jz = j;
#pragma unroll
        for (int j = 0; j < 4; ++j) r.u[j] = (j == jz) ? 1.0f : 0.0f;
        r.Ji = 0.0f;
        r.K = 0.0f;
    }
    return r;
}

// Eq. 3 / Eq. 1 partial sums of one voxel.
template <int C, bool M2>
__device__ __forceinline__ void memb_accumulate(const Memb &r, float xv, float m, float2 (&num2)[2],
                                                float2 (&den2)[2], float &Jacc) {
    constexpr int NP = (C + 1) / 2;
    const float2 x2 = make_float2(xv, xv);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const float2 uu = make_float2(r.u[2 * q], r.u[2 * q + 1]);
        float2 um;
        if (M2) {
            um = __fmul2_rn(uu, uu);
        } else {
            um.x = uu.x > 0.f ? exp2f(m * log2f(uu.x)) : 0.f;
            um.y = uu.y > 0.f ? exp2f(m * log2f(uu.y)) : 0.f;
        }
        num2[q] = __ffma2_rn(um, x2, num2[q]);  // Eq. 3 numerator
        den2[q] = __fadd2_rn(den2[q], um);      // Eq. 3 denominator
    }
    Jacc += r.Ji;
}

template <int C, bool M2>
__device__ __forceinline__ float4 membership2(float xv, const float2 (&c2)[2], const float2 (&A)[2], float m,
                                              float inv_m1, float2 (&num2)[2], float2 (&den2)[2],
                                              float &Jacc) {
    const Memb r = memb_compute<C, M2>(xv, c2, A, m, inv_m1, A);
    memb_accumulate<C, M2>(r, xv, m, num2, den2, Jacc);
    return make_float4(r.u[0], r.u[1], r.u[2], r.u[3]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

}  // namespace pifcm
