// fcm_hist.cu -- the FCM start of a quantised (u8 / u16) volume on its value
// histogram (Alg. 1 step 2; Alg. 2 step 5,
// FCM = the IFCM step with lambda = xi = 0).
//
// With lambda = xi = 0 the Eq. 4 factor is 1, so d2_ij = (x_i - c_j)^2 and the
// Eq. 2 memberships of voxel i depend on x_i and the centres only: all voxels
// of one intensity value get the same row.  The Eq. 3 sums (sum u^m x,
// sum u^m), the Eq. 1 cost and max |u_new - u_old| over the voxels therefore
// equal the count-weighted sums (and the max) over the distinct values.  The
// whole FCM loop runs on <= 65536 values in one CTA; the voxels' memberships
// are written once, at the end, from the centres of the last iteration
// (k_fcm_memberships, one pass over x).  Both kernels evaluate a row with the
// same device function (`membership`, step_common.cuh) on the same fp32
// x = normalize_q(v) as k_normalize, so a voxel's written row is bit-identical
// to the row its value contributed to the sums.
#include <cuda_runtime.h>
#include <math.h>

#include "pifcm_internal.cuh"
#include "step_common.cuh"

namespace pifcm {

constexpr int kFhThreads = 1024;
constexpr int kFhWarps = kFhThreads / 32;

// counts[v] += #voxels with value v (u8: 256 entries, shared-memory bins;
// u16: 65536 entries, global atomics).
__global__ void k_value_hist_u8(const uint8_t *vol, long long n, int64_t *counts) {
    __shared__ unsigned int h[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        atomicAdd(&h[vol[i]], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd((unsigned long long *)&counts[b], (unsigned long long)h[b]);
}
__global__ void k_value_hist_u16(const uint16_t *vol, long long n, int64_t *counts) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&counts[vol[i]], 1ull);
}

cudaError_t launch_value_hist(const void *vol, int dtype, long long n, int64_t *counts, cudaStream_t st) {
    long long b = (n + 256 * 32 - 1) / (256 * 32);
    if (b > 148 * 4) b = 148 * 4;
    if (b < 1) b = 1;
    if (dtype == PIFCM_U8)
        k_value_hist_u8<<<(int)b, 256, 0, st>>>(static_cast<const uint8_t *>(vol), n, counts);
    else if (dtype == PIFCM_U16)
        k_value_hist_u16<<<(int)b, 256, 0, st>>>(static_cast<const uint16_t *>(vol), n, counts);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// One CTA.  (1) the occupied values in ascending order -> xs (their x),
// ns (their counts); (2) FCM iterations t = 1..max_iter: memberships of every
// value at the current centres, count-weighted fp64 sums in a fixed order
// (per-thread strided sums, xor-shuffle trees, warps in index order), Eq. 3
// centres (kept if sum u^m < 1e-12, R9), Eq. 1 cost, max |du| (t = 1: 1, R14),
// stop when max |du| < eps.
template <int C, bool M2>
__global__ void __launch_bounds__(kFhThreads) k_fcm_hist(FcmHistArgs a) {
    __shared__ int s_scan[kFhWarps];
    __shared__ int s_base, s_stop;
    __shared__ float s_c[kMaxC];
    __shared__ double red[kFhWarps][kNR];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lo = (int)a.mm[0], hi = (int)a.mm[1];
    if (tid == 0) { s_base = 0; s_stop = 0; }
    if (tid < kMaxC) s_c[tid] = a.c0[tid];
    __syncthreads();
    // (1) stream compaction of the occupied values (block-wide exclusive scan)
    for (int v0 = 0; v0 < a.nvals; v0 += kFhThreads) {
        const int v = v0 + tid;
        const long long cnt = v < a.nvals ? (long long)a.counts[v] : 0;
        const int f = cnt > 0 ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_scan[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            const int w = s_scan[lane];
            int incl = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            s_scan[lane] = incl - w;
        }
        __syncthreads();
        const int pos = s_base + s_scan[warp] + __popc(bal & ((1u << lane) - 1u));
        if (f) {
            a.xs[pos] = normalize_q(v, lo, hi);  // Alg. 2 step 1, the x of k_normalize
            a.ns[pos] = (double)cnt;
        }
        __syncthreads();
        if (tid == kFhThreads - 1) s_base = pos + f;
        __syncthreads();
    }
    const int nocc = s_base;
    const float ones[kMaxC] = {1.f, 1.f, 1.f, 1.f};  // lambda = xi = 0: Eq. 4 factor 1
    int t;
    double J = 0.0, du = 0.0;
    for (t = 1; t <= a.max_iter; ++t) {
        float c[kMaxC];
#pragma unroll
        for (int j = 0; j < kMaxC; ++j) c[j] = s_c[j];
        double v[kNR];
#pragma unroll
        for (int r = 0; r < kNR; ++r) v[r] = 0.0;
        for (int k = tid; k < nocc; k += kFhThreads) {
            float nf[kMaxC] = {0.f, 0.f, 0.f, 0.f}, df[kMaxC] = {0.f, 0.f, 0.f, 0.f}, Jf = 0.f;
            const float4 u = membership<C, M2>(a.xs[k], c, ones, a.m, a.inv_m1, nf, df, Jf);  // Eq. 2
            const double n = a.ns[k];
#pragma unroll
            for (int j = 0; j < C; ++j) {
                v[j] += n * (double)nf[j];           // Eq. 3 numerator: u^m x of the value
                v[kMaxC + j] += n * (double)df[j];   // Eq. 3 denominator: u^m
            }
            v[2 * kMaxC] += n * (double)Jf;          // Eq. 1
            if (t > 1) {
                const float4 o = a.up[k];
                const float d = fmaxf(fmaxf(fabsf(u.x - o.x), fabsf(u.y - o.y)),
                                      fmaxf(fabsf(u.z - o.z), fabsf(u.w - o.w)));
                v[kNR - 1] = fmax(v[kNR - 1], (double)d);
            }
            a.up[k] = u;
        }
#pragma unroll
        for (int r = 0; r < kNR; ++r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double q = __shfl_xor_sync(0xffffffffu, v[r], o);
                v[r] = (r == kNR - 1) ? fmax(v[r], q) : v[r] + q;
            }
        }
        if (lane == 0)
#pragma unroll
            for (int r = 0; r < kNR; ++r) red[warp][r] = v[r];
        __syncthreads();
        if (tid == 0) {
            double s[kNR];
#pragma unroll
            for (int r = 0; r < kNR; ++r) s[r] = red[0][r];
            for (int w = 1; w < kFhWarps; ++w)
#pragma unroll
                for (int r = 0; r < kNR; ++r) s[r] = (r == kNR - 1) ? fmax(s[r], red[w][r]) : s[r] + red[w][r];
            for (int j = 0; j < kMaxC; ++j) a.c_prev[j] = c[j];  // the centres this iteration's rows used
            for (int j = 0; j < C; ++j)
                if (s[kMaxC + j] >= kDenEps) s_c[j] = (float)(s[j] / s[kMaxC + j]);  // Eq. 3, R9
            J = s[2 * kMaxC];
            du = (t == 1) ? 1.0 : s[kNR - 1];  // R14: the first iteration never stops
            s_stop = (a.eps > 0.f && du < (double)a.eps) ? 1 : 0;
        }
        __syncthreads();
        if (s_stop) break;
    }
    if (tid == 0) {
        for (int j = 0; j < kMaxC; ++j) a.c_out[j] = s_c[j];
        const int done = t > a.max_iter ? a.max_iter : t;
        a.stats[0] = J;
        a.stats[1] = du;
        a.stats[2] = (double)done;
        a.stats[3] = s_stop ? 1.0 : 0.0;
        if (!isfinite(J) && a.status) atomicExch(a.status, (int)PIFCM_ENUMERIC);
    }
}

cudaError_t launch_fcm_hist(const FcmHistArgs &a, int C, bool m2, cudaStream_t st) {
#define PIFCM_FH(CC)                                                               \
    if (m2)                                                                        \
        k_fcm_hist<CC, true><<<1, kFhThreads, 0, st>>>(a);                         \
    else                                                                           \
        k_fcm_hist<CC, false><<<1, kFhThreads, 0, st>>>(a);
    switch (C) {
        case 2: PIFCM_FH(2) break;
        case 3: PIFCM_FH(3) break;
        case 4: PIFCM_FH(4) break;
        default: return cudaErrorInvalidValue;
    }
#undef PIFCM_FH
    return cudaGetLastError();
}

// U_i = Eq. 2 memberships of x_i at the centres c (lambda = xi = 0), every
// voxel of the grid: x [nz][ny][pitch] -> U [nz][ny][nx][4].
template <int C, bool M2>
__global__ void k_fcm_memberships(const float *x, int nx, long long nvox, int pitch, const float *cen, float m,
                                  float inv_m1, float4 *U) {
    float c[kMaxC];
#pragma unroll
    for (int j = 0; j < kMaxC; ++j) c[j] = cen[j];
    const float ones[kMaxC] = {1.f, 1.f, 1.f, 1.f};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nvox;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / nx;
        float nf[kMaxC] = {0.f, 0.f, 0.f, 0.f}, df[kMaxC] = {0.f, 0.f, 0.f, 0.f}, Jf = 0.f;
        const float xv = x[row * pitch + (i - row * nx)];
        __stcs(U + i, membership<C, M2>(xv, c, ones, m, inv_m1, nf, df, Jf));
    }
}

cudaError_t launch_fcm_memberships(const float *x, int nx, int ny, int nz, int pitch, const float *c, int C,
                                   float m, float4 *U, cudaStream_t st) {
    const long long nvox = (long long)nx * ny * nz;
    long long b = (nvox + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    if (b < 1) b = 1;
    const bool m2 = (m == 2.0f);
    const float inv_m1 = 1.0f / (m - 1.0f);
#define PIFCM_FM(CC)                                                                                      \
    if (m2)                                                                                               \
        k_fcm_memberships<CC, true><<<(int)b, 256, 0, st>>>(x, nx, nvox, pitch, c, m, inv_m1, U);         \
    else                                                                                                  \
        k_fcm_memberships<CC, false><<<(int)b, 256, 0, st>>>(x, nx, nvox, pitch, c, m, inv_m1, U);
    switch (C) {
        case 2: PIFCM_FM(2) break;
        case 3: PIFCM_FM(3) break;
        case 4: PIFCM_FM(4) break;
        default: return cudaErrorInvalidValue;
    }
#undef PIFCM_FM
    return cudaGetLastError();
}

}  // namespace pifcm
