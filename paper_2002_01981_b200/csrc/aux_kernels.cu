// aux_kernels.cu -- everything on the path except the fused step: the Eq. 3 /
// Eq. 1 finalisation, the device PSO (Alg. 1 steps 3-8), normalisation and
// histogram (Alg. 2 step 1), the GMM start (R15), defuzzification.
#include <cuda_runtime.h>
#include <math.h>

#include "pifcm_internal.cuh"

namespace pifcm {

// ---------------------------------------------------------------- finalize
// Eq. 3 c_j = sum u^m x / sum u^m (keep c_j if the sum < 1e-12,
// R9) and Eq. 1 J from per-chunk fp64 partial records.  One CTA
// is finalised by the last step CTA itself (finalize_if_last in step.cu);
// the z-slab records gathered across ranks by k_slab_finalize below, with
// the same thread count and summation order, so the single-GPU canonical
// run and any slab split give bit-identical centres and J.
constexpr int kFinThreads = kStepThreads;

// After an early-converged pifcm_iterate: the last U of state p was written
// by iteration stats[p][2]; iterations t with (iters - t) odd wrote to the
// scratch buffer, so those states are copied to U_out.
__global__ void k_fixup_copy(const float4 *scratch, float4 *out, long long nvox, int iters,
                             const double *stats) {
    const int p = blockIdx.y;
    const int done = (int)stats[4 * p + 2];
    if (((iters - done) & 1) == 0) return;
    const float4 *s = scratch + (long long)p * nvox;
    float4 *o = out + (long long)p * nvox;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nvox;
         i += (long long)gridDim.x * blockDim.x)
        o[i] = s[i];
}

cudaError_t launch_fixup_copy(const float4 *scratch, float4 *out, long long nvox, int P,
                              const double *stats, int iters, cudaStream_t st) {
    dim3 grid(148 * 4, P);
    k_fixup_copy<<<grid, 256, 0, st>>>(scratch, out, nvox, iters, stats);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- z-slab
// Records of all ranks, gathered [world][P][nrec][kNR] (rank w holds
// counts[w] <= nrec real records, the rest is padding), summed for state p in
// canonical order -- rank-major, record-minor over the real records only,
// which is the global z-chunk order and the same sequence for any number of
// slabs -- then Eq. 3 / Eq. 1.  The thread assignment depends only on the
// canonical index, so the fp64 result is identical for any slab count.
__global__ void __launch_bounds__(kFinThreads) k_slab_finalize(int C, int P, int world, int nrec,
                                                             const int *counts, const double *rec,
                                                             float *centers, double *stats, double *fitness,
                                                             float eps, int *status) {
    __shared__ double red[kFinThreads][kNR];
    __shared__ int cnt[64];
    const int p = blockIdx.x;
    if (stats && stats[4 * p + 3] != 0.0) return;
    for (int w = threadIdx.x; w < world && w < 64; w += blockDim.x) cnt[w] = counts ? counts[w] : nrec;
    __syncthreads();
    long long total = 0;
    for (int w = 0; w < world; ++w) total += cnt[w];
    double v[kNR];
#pragma unroll
    for (int r = 0; r < kNR; ++r) v[r] = 0.0;
    int w = 0;
    long long base = 0;  // canonical index of rank w's first record
    for (long long c = threadIdx.x; c < total; c += kFinThreads) {
        while (c >= base + cnt[w]) {
            base += cnt[w];
            ++w;
        }
        const double *src = rec + (((long long)w * P + p) * nrec + (c - base)) * kNR;
#pragma unroll
        for (int r = 0; r < kNR - 1; ++r) v[r] += src[r];
        v[kNR - 1] = fmax(v[kNR - 1], src[kNR - 1]);
    }
#pragma unroll
    for (int r = 0; r < kNR; ++r) red[threadIdx.x][r] = v[r];
    __syncthreads();
    for (int s = kFinThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
#pragma unroll
            for (int r = 0; r < kNR - 1; ++r) red[threadIdx.x][r] += red[threadIdx.x + s][r];
            red[threadIdx.x][kNR - 1] = fmax(red[threadIdx.x][kNR - 1], red[threadIdx.x + s][kNR - 1]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double J = red[0][2 * kMaxC], du = red[0][2 * kMaxC + 1];
        for (int j = 0; j < C; ++j) {
            const double num = red[0][j], den = red[0][kMaxC + j];
            if (den >= kDenEps) centers[4 * p + j] = (float)(num / den);
        }
        if (fitness) fitness[p] = J;
        if (stats) {
            stats[4 * p + 0] = J;
            stats[4 * p + 1] = du;
            stats[4 * p + 2] += 1.0;
            stats[4 * p + 3] = (eps > 0.f && du < (double)eps) ? 1.0 : 0.0;
        }
        if (!isfinite(J) && status) atomicExch(status, (int)PIFCM_ENUMERIC);
    }
}

cudaError_t launch_slab_finalize(int C, int P, int world, int nrec, const int *counts, const double *records,
                                 float *centers, double *stats, double *fitness, float eps, int *status,
                                 cudaStream_t st) {
    if (world > 64) return cudaErrorInvalidValue;
    k_slab_finalize<<<P, kFinThreads, 0, st>>>(C, P, world, nrec, counts, records, centers, stats, fitness, eps,
                                               status);
    return cudaGetLastError();
}

// Copy one plane of every state between a slab array and a packed buffer
// (halo pack / unpack), or zero it (a halo outside the volume).
__global__ void k_halo_copy(const float4 *src, long long src_state, float4 *dst, long long dst_state,
                            long long plane, bool zero, const int *src_idx, const int *dst_idx) {
    const int p = blockIdx.y;
    const long long so = (long long)(src_idx ? src_idx[p] : p) * src_state;
    const long long dof = (long long)(dst_idx ? dst_idx[p] : p) * dst_state;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (long long)gridDim.x * blockDim.x)
        dst[dof + i] = zero ? make_float4(0.f, 0.f, 0.f, 0.f) : src[so + i];
}

cudaError_t launch_halo_copy(const float4 *src, long long src_state, float4 *dst, long long dst_state,
                             long long plane, int P, bool zero, cudaStream_t st, const int *src_idx,
                             const int *dst_idx) {
    long long b = (plane + 255) / 256;
    if (b > 148 * 4) b = 148 * 4;
    dim3 grid((unsigned)(b < 1 ? 1 : b), P);
    k_halo_copy<<<grid, 256, 0, st>>>(src, src_state, dst, dst_state, plane, zero, src_idx, dst_idx);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al. SC'11), the counter-based generator shared by
// specification (not code) with the oracle so both see the same draws (R12).
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c[0];
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// Two uniform doubles in [0,1) (53 bits each) for counter (c0, c1, c2, 0).
__device__ __forceinline__ void draw2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t k0,
                                      uint32_t k1, double &a, double &b) {
    uint32_t c[4] = {c0, c1, c2, 0u};
    philox4x32_10(c, k0, k1);
    const unsigned long long wa = ((unsigned long long)c[1] << 32) | c[0];
    const unsigned long long wb = ((unsigned long long)c[3] << 32) | c[2];
    a = (double)(wa >> 11) * (1.0 / 9007199254740992.0);
    b = (double)(wb >> 11) * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------- PSO init
// Alg. 1 step 3: positions ~ U[0,1]^2 from counter
// (0xFFFFFFFF, p, 1, 0), velocities ~ U[-v0, v0]^2 from (0xFFFFFFFF, p, 2, 0)
// (R12).  Every local particle's state is slot 0 (the start state); the first
// evaluation of local particle q writes slot 1 + q.
__global__ void k_pso_init(SwarmDev s, int P, int Pl, int p0, double v0, uint32_t k0,
                           uint32_t k1, const float *c0, int nslots) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        double a, b;
        draw2(0xFFFFFFFFu, (uint32_t)p, 1u, k0, k1, a, b);
        s.pos[2 * p] = a;
        s.pos[2 * p + 1] = b;
        draw2(0xFFFFFFFFu, (uint32_t)p, 2u, k0, k1, a, b);
        s.vel[2 * p] = __dmul_rn(__dsub_rn(__dmul_rn(2.0, a), 1.0), v0);
        s.vel[2 * p + 1] = __dmul_rn(__dsub_rn(__dmul_rn(2.0, b), 1.0), v0);
        s.pbf[p] = INFINITY;
        s.pbx[2 * p] = s.pos[2 * p];
        s.pbx[2 * p + 1] = s.pos[2 * p + 1];
        s.fit[p] = INFINITY;
    }
    for (int q = threadIdx.x; q < Pl; q += blockDim.x) {
        s.cur[q] = 0;
        s.nxt[q] = 1 + q;
        for (int j = 0; j < kMaxC; ++j) s.centers[4 * q + j] = c0[j];
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) s.hdr[i] = 0;
        s.hdr[kHGbest] = -1;
        s.hdr[kHGbestSlot] = -1;
        s.hdr[kHInit] = 1;
        for (int i = 0; i < 16; ++i) s.dhdr[i] = 0.0;  // the whole record is read back (pifcm_pso_result_get)
        s.dhdr[kDPrevGf] = INFINITY;
        s.dhdr[kDGbestJ] = INFINITY;
        s.dhdr[kDGbestL] = 0.0;
        s.dhdr[kDGbestX] = 0.0;
        for (int j = 0; j < kMaxC; ++j) s.gbest_c[j] = c0[j];
    }
    (void)nslots;
}

cudaError_t launch_pso_init(SwarmDev s, int P, int Pl, int p0, double v0, uint32_t k0,
                            uint32_t k1, const float *c0, int nslots, cudaStream_t st) {
    k_pso_init<<<1, 256, 0, st>>>(s, P, Pl, p0, v0, k0, k1, c0, nslots);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- PSO update
// After the fitnesses f[P] of generation t (evaluated at s.pos) are known:
//   step 5:  pbest, strict <
//   gbest = argmin pbest (lowest index on ties); on a strict improvement the
//           gbest snapshot (Alg. 1 step 10) = the state that
//           particle's evaluation produced (its new slot), pinned
//   step 6: lbest over the ring {p-k..p+k} mod P (R12)
//   step 7: v += p1 (pbest - x) + p2 (lbest - x), |v| <= vmax, with
//           (p1, p2) from Philox counter (t, p, 0, 0)
//   step 8: x = clamp(x + v, 0, 1)
//   step 9: calm generations counter and stop flag (R12)
// Slots: each local particle's new state is in nxt[q] -> becomes cur[q]; the
// next evaluation writes to the lowest-numbered slots that are neither a
// current state nor the pinned gbest (2*Pl + 1 slots always suffice).
constexpr int kPsoThreads = 256;

__global__ void __launch_bounds__(kPsoThreads) k_pso_update(const PsoUpdateArgs a) {
    SwarmDev s = a.s;
    __shared__ int lb_sh[1024];
    if (s.hdr[kHStop]) return;
    const int t = s.hdr[kHGen];
    // step 5 (and remember the evaluation positions)
    for (int p = threadIdx.x; p < a.P; p += blockDim.x) {
        s.evalpos[2 * p] = s.pos[2 * p];
        s.evalpos[2 * p + 1] = s.pos[2 * p + 1];
        const double f = s.fit[p];
        if (a.tr_f && t < a.tr_max) {
            a.tr_f[(long long)t * a.P + p] = f;
            a.tr_pos[2 * ((long long)t * a.P + p)] = s.pos[2 * p];
            a.tr_pos[2 * ((long long)t * a.P + p) + 1] = s.pos[2 * p + 1];
        }
        if (f < s.pbf[p]) {
            s.pbf[p] = f;
            s.pbx[2 * p] = s.pos[2 * p];
            s.pbx[2 * p + 1] = s.pos[2 * p + 1];
        }
    }
    __syncthreads();
    // step 6: ring lbest
    for (int p = threadIdx.x; p < a.P; p += blockDim.x) {
        int best = -1;
        for (int d = -a.ring_k; d <= a.ring_k; ++d) {
            const int q = ((p + d) % a.P + a.P) % a.P;
            if (best < 0 || s.pbf[q] < s.pbf[best] || (s.pbf[q] == s.pbf[best] && q < best))
                best = q;
        }
        lb_sh[p] = best;
    }
    if (threadIdx.x == 0) {
        // gbest, snapshot, slots, stop rule
        int g = 0;
        for (int p = 1; p < a.P; ++p)
            if (s.pbf[p] < s.pbf[g]) g = p;
        // R13: on an exact tie the incumbent keeps the gbest (its state is the
        // pinned snapshot, so gbest_particle always names the snapshot's owner)
        const int g_old = s.hdr[kHGbest];
        if (g_old >= 0 && !(s.pbf[g] < s.pbf[g_old])) g = g_old;
        const double gf_old = s.dhdr[kDGbestJ];
        const int improved = (s.pbf[g] < gf_old) ? 1 : 0;
        s.hdr[kHGbest] = g;
        if (a.tr_gbest && t < a.tr_max) a.tr_gbest[t] = g;
        if (a.mode == PIFCM_FIT_CHAINED) {
            for (int q = 0; q < a.Pl; ++q) s.cur[q] = s.nxt[q];
            if (improved) {
                s.dhdr[kDGbestJ] = s.pbf[g];
                s.dhdr[kDGbestL] = s.pos[2 * g];
                s.dhdr[kDGbestX] = s.pos[2 * g + 1];
                const int gl = g - a.p0;
                if (gl >= 0 && gl < a.Pl) {
                    s.hdr[kHGbestSlot] = s.cur[gl];
                    for (int j = 0; j < kMaxC; ++j) s.gbest_c[j] = s.centers[4 * gl + j];
                } else {
                    s.hdr[kHGbestSlot] = -1;
                }
            }
            // free-slot assignment for the next evaluation (batched: per batch,
            // by k_assign_batch before each evaluation launch)
            if (!a.batched) {
                unsigned int used[(2 * 1024 + 1 + 31) / 32];
                const int nw = (a.nslots + 31) / 32;
                for (int w = 0; w < nw; ++w) used[w] = 0u;
                for (int q = 0; q < a.Pl; ++q) used[s.cur[q] >> 5] |= 1u << (s.cur[q] & 31);
                const int gs = s.hdr[kHGbestSlot];
                if (gs >= 0) used[gs >> 5] |= 1u << (gs & 31);
                int next_free = 0;
                for (int q = 0; q < a.Pl; ++q) {
                    while (used[next_free >> 5] & (1u << (next_free & 31))) ++next_free;
                    s.nxt[q] = next_free++;
                }
            }
        } else {
            // ANCHORED: slot 0 = the shared start, slot 1 = the gbest snapshot
            // (written by the guarded snapshot step after this kernel).
            // LEADER: three slots: the shared state cur[0], the slot nxt[0] the
            // advance writes, and the pinned gbest snapshot.
            if (improved) {
                s.dhdr[kDGbestJ] = s.pbf[g];
                s.dhdr[kDGbestL] = s.pos[2 * g];
                s.dhdr[kDGbestX] = s.pos[2 * g + 1];
            }
            if (a.mode == PIFCM_FIT_LEADER) {
                int nf = 0;
                while (nf == s.cur[0] || nf == s.hdr[kHGbestSlot]) ++nf;
                s.nxt[0] = nf;
                if (improved) s.hdr[kHGbestSlot] = nf;
            } else if (improved) {
                s.hdr[kHGbestSlot] = 1;
            }
        }
        s.hdr[kHImproved] = improved;
        s.hdr[kHNotImproved] = improved ? 0 : 1;
        // step 9 stop rule on the relative decrease of the gbest fitness
        const double gf = s.pbf[g];
        if (t > 0 && a.patience > 0) {
            const double rel = __ddiv_rn(__dsub_rn(s.dhdr[kDPrevGf], gf), (gf > 0.0 ? gf : 1.0));
            s.hdr[kHCalm] = (rel < a.tol) ? s.hdr[kHCalm] + 1 : 0;
            if (s.hdr[kHCalm] >= a.patience) s.hdr[kHStop] = 1;
        }
        s.dhdr[kDPrevGf] = gf;
        s.hdr[kHGen] = t + 1;
    }
    __syncthreads();
    // steps 7-8
    for (int p = threadIdx.x; p < a.P; p += blockDim.x) {
        double p1, p2;
        draw2((uint32_t)t, (uint32_t)p, 0u, a.key0, a.key1, p1, p2);
        const int lb = lb_sh[p];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            // explicit roundings (no FMA contraction): the same fp64 operations,
            // in the same order, as the written formula
            const double x = s.pos[2 * p + d];
            const double t1 = __dmul_rn(p1, __dsub_rn(s.pbx[2 * p + d], x));
            const double t2 = __dmul_rn(p2, __dsub_rn(s.pbx[2 * lb + d], x));
            double v = __dadd_rn(__dadd_rn(s.vel[2 * p + d], t1), t2);
            v = fmin(fmax(v, -a.vmax), a.vmax);
            s.vel[2 * p + d] = v;
            s.pos[2 * p + d] = fmin(fmax(__dadd_rn(x, v), 0.0), 1.0);
        }
    }
}

// Batched CHAINED evaluation (pifcm_pso_cfg.eval_batch): before the launch of
// local particles [b0, b0 + nb), their output slots = the lowest slots that
// hold no live state: live = the new states of the particles evaluated
// earlier in this generation (nxt[q], q < b0), the current states of the rest
// (cur[q], q >= b0) and the pinned gbest snapshot -- at most Pl + 1 slots, so
// Pl + nb + 1 slots always suffice.
__global__ void k_assign_batch(SwarmDev s, int Pl, int b0, int nb, int nslots) {
    if (threadIdx.x != 0 || s.hdr[kHStop]) return;
    unsigned int used[(2 * 1024 + 1 + 31) / 32];
    const int nw = (nslots + 31) / 32;
    for (int w = 0; w < nw; ++w) used[w] = 0u;
    for (int q = 0; q < Pl; ++q) {
        const int sl = q < b0 ? s.nxt[q] : s.cur[q];
        used[sl >> 5] |= 1u << (sl & 31);
    }
    const int gs = s.hdr[kHGbestSlot];
    if (gs >= 0) used[gs >> 5] |= 1u << (gs & 31);
    int next_free = 0;
    for (int q = b0; q < b0 + nb; ++q) {
        while (used[next_free >> 5] & (1u << (next_free & 31))) ++next_free;
        s.nxt[q] = next_free++;
    }
}
cudaError_t launch_assign_batch(SwarmDev s, int Pl, int b0, int nb, int nslots, cudaStream_t st) {
    k_assign_batch<<<1, 32, 0, st>>>(s, Pl, b0, nb, nslots);
    return cudaGetLastError();
}

cudaError_t launch_pso_update(const PsoUpdateArgs &a, cudaStream_t st) {
    k_pso_update<<<1, kPsoThreads, 0, st>>>(a);
    return cudaGetLastError();
}

// gbest (lambda*, xi*) -> a [1][2] lam_xi buffer for the final IFCM.
__global__ void k_set_lamxi(double *dst, const double *dhdr) {
    dst[0] = dhdr[kDGbestL];
    dst[1] = dhdr[kDGbestX];
}
cudaError_t launch_set_lamxi(double *dst, const double *dhdr, cudaStream_t st) {
    k_set_lamxi<<<1, 1, 0, st>>>(dst, dhdr);
    return cudaGetLastError();
}

// Copy the pinned gbest slot to U_out and its centres to c_out.
__global__ void k_gather_gbest(const float4 *slots, long long nvox, const int *hdr,
                               const float *gbest_c, float4 *U_out, float *c_out) {
    const int gs = hdr[kHGbestSlot];
    if (gs < 0) return;
    const float4 *src = slots + (long long)gs * nvox;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nvox;
         i += (long long)gridDim.x * blockDim.x)
        U_out[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x < kMaxC && c_out) c_out[threadIdx.x] = gbest_c[threadIdx.x];
}
cudaError_t launch_gather_gbest(const float4 *slots, long long nvox, const int *hdr,
                                const float *gbest_c, float4 *U_out, float *c_out,
                                cudaStream_t st) {
    k_gather_gbest<<<148 * 4, 256, 0, st>>>(slots, nvox, hdr, gbest_c, U_out, c_out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- normalise
// Alg. 2 step 1 for u8 / u16 / f32 volumes.
// min / max are reduced as order-preserving 32-bit keys: the value itself for
// the unsigned types, the sign-flipped bit pattern for floats.
__device__ __forceinline__ unsigned key_of(uint8_t v) { return v; }
__device__ __forceinline__ unsigned key_of(uint16_t v) { return v; }
__device__ __forceinline__ unsigned key_of(float v) {
    const unsigned b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ double value_of_key(unsigned k, int dtype) {
    if (dtype != PIFCM_F32) return (double)k;
    const unsigned b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    return (double)__uint_as_float(b);
}

template <typename T>
__global__ void k_minmax(const T *vol, long long n, unsigned int *mm) {
    unsigned int lo = 0xFFFFFFFFu, hi = 0u;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned int v = key_of(vol[i]);
        lo = min(lo, v);
        hi = max(hi, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}
__global__ void k_mm_reset(unsigned int *mm) {
    mm[0] = 0xFFFFFFFFu;
    mm[1] = 0u;
}
template <typename T>
static cudaError_t launch_minmax_t(const T *vol, long long n, unsigned int *mm, cudaStream_t st) {
    k_mm_reset<<<1, 1, 0, st>>>(mm);
    long long b = (n + 256 * 16 - 1) / (256 * 16);
    if (b > 148 * 8) b = 148 * 8;
    if (b < 1) b = 1;
    k_minmax<T><<<(int)b, 256, 0, st>>>(vol, n, mm);
    return cudaGetLastError();
}

// x = (v - min) / (max - min), constant volume -> 0 (R16), pitched rows.
// u8 / u16: exact integer differences, one correctly rounded fp32 division;
// f32: the quotient in fp64, rounded once to fp32.
template <typename T>
__global__ void k_normalize(const T *vol, int nx, int ny, int nz, int pitch, const unsigned int *mm, float *x,
                            int dtype) {
    const double lo = value_of_key(mm[0], dtype), hi = value_of_key(mm[1], dtype);
    const long long rows = (long long)ny * nz;
    const long long n = rows * pitch;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const long long row = e / pitch;
        const int X = (int)(e - row * pitch);
        float v = 0.f;
        if (X < nx && hi > lo) {
            const T t = vol[row * nx + X];
            if (dtype == PIFCM_F32)
                v = (float)(((double)t - lo) / (hi - lo));
            else
                v = normalize_q((int)t, (int)lo, (int)hi);
        }
        x[e] = v;
    }
}

// R15: 256-bin histogram.  u8 / u16 in integers:
// bin = ((v-min)*255 + (max-min)/2) / (max-min); f32 in fp64:
// bin = floor((v-min)*255/(max-min) + 0.5) (the oracle's arithmetic).
template <typename T>
__global__ void k_hist(const T *vol, long long n, const unsigned int *mm, int64_t *hist, int dtype) {
    __shared__ unsigned int h[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0u;
    __syncthreads();
    const double lo = value_of_key(mm[0], dtype), hi = value_of_key(mm[1], dtype);
    const long long ilo = (long long)lo, irng = (long long)hi - (long long)lo;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int b = 0;
        if (hi > lo) {
            if (dtype == PIFCM_F32) {
                b = (int)floor(((double)vol[i] - lo) * 255.0 / (hi - lo) + 0.5);
                b = min(max(b, 0), 255);
            } else {
                b = (int)((((long long)vol[i] - ilo) * 255 + irng / 2) / irng);
            }
        }
        atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd((unsigned long long *)&hist[b], (unsigned long long)h[b]);
}
__global__ void k_zero_i64(int64_t *p, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

cudaError_t launch_minmax(const void *vol, int dtype, long long n, unsigned int *mm, cudaStream_t st) {
    switch (dtype) {
        case PIFCM_U8: return launch_minmax_t(static_cast<const uint8_t *>(vol), n, mm, st);
        case PIFCM_U16: return launch_minmax_t(static_cast<const uint16_t *>(vol), n, mm, st);
        case PIFCM_F32: return launch_minmax_t(static_cast<const float *>(vol), n, mm, st);
        default: return cudaErrorInvalidValue;
    }
}
cudaError_t launch_normalize(const void *vol, int dtype, int nx, int ny, int nz, int pitch,
                             const unsigned int *mm, float *x, cudaStream_t st) {
    switch (dtype) {
        case PIFCM_U8: k_normalize<<<148 * 8, 256, 0, st>>>(static_cast<const uint8_t *>(vol), nx, ny, nz, pitch, mm, x, dtype); break;
        case PIFCM_U16: k_normalize<<<148 * 8, 256, 0, st>>>(static_cast<const uint16_t *>(vol), nx, ny, nz, pitch, mm, x, dtype); break;
        case PIFCM_F32: k_normalize<<<148 * 8, 256, 0, st>>>(static_cast<const float *>(vol), nx, ny, nz, pitch, mm, x, dtype); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
cudaError_t launch_hist(const void *vol, int dtype, long long n, const unsigned int *mm, int64_t *hist,
                        cudaStream_t st) {
    k_zero_i64<<<1, 256, 0, st>>>(hist, 256);
    long long b = (n + 256 * 32 - 1) / (256 * 32);
    if (b > 148 * 4) b = 148 * 4;
    if (b < 1) b = 1;
    switch (dtype) {
        case PIFCM_U8: k_hist<<<(int)b, 256, 0, st>>>(static_cast<const uint8_t *>(vol), n, mm, hist, dtype); break;
        case PIFCM_U16: k_hist<<<(int)b, 256, 0, st>>>(static_cast<const uint16_t *>(vol), n, mm, hist, dtype); break;
        case PIFCM_F32: k_hist<<<(int)b, 256, 0, st>>>(static_cast<const float *>(vol), n, mm, hist, dtype); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
cudaError_t launch_minmax_u8(const uint8_t *vol, long long n, unsigned int *mm, cudaStream_t st) {
    return launch_minmax(vol, PIFCM_U8, n, mm, st);
}
cudaError_t launch_normalize_u8(const uint8_t *vol, int nx, int ny, int nz, int pitch, const unsigned int *mm,
                                float *x, cudaStream_t st) {
    return launch_normalize(vol, PIFCM_U8, nx, ny, nz, pitch, mm, x, st);
}
cudaError_t launch_hist_u8(const uint8_t *vol, long long n, const unsigned int *mm, int64_t *hist,
                           cudaStream_t st) {
    return launch_hist(vol, PIFCM_U8, n, mm, hist, st);
}

// ---------------------------------------------------------------- GMM start
// R15 ("Modified_FCM with Gaussian mixture model"): 1-D EM of a
// C-component mixture on the 256-bin histogram, bin b at level b/255; start
// mu_j = (j+0.5)/C, sigma_j^2 = 1/(4C^2), w_j = 1/C; variance floor 1e-6;
// stop when no mean moves by 1e-9 or after max_iter; means sorted ascending;
// fewer than C occupied bins or coincident means -> c_j = j/(C-1).
// One block, one thread per bin, fp64; every reduction is a fixed-order
// xor-shuffle tree inside each warp followed by the 8 warp results in order,
// all statistics of a pass reduced together (two passes per EM iteration).
template <int NV>
__device__ __forceinline__ void block_sum_vec(double (&v)[NV], double (*sh)[NV]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[warp][i] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double t = sh[0][i];
        for (int w = 1; w < 8; ++w) t += sh[w][i];
        v[i] = t;
    }
    __syncthreads();
}

// C is a template parameter so that the per-component work of a bin (the
// exp, the normalisation, the moments) is unrolled: the C chains run
// interleaved instead of back to back (the loop is latency-bound, one block).
template <int C>
__global__ void __launch_bounds__(256) k_gmm(const int64_t *hist, int max_iter, float *c0) {
    __shared__ double sh1[8][2 * kMaxC + 2];
    __shared__ double sh2[8][kMaxC];
    double mu[C], s2[C], w[C];
    const int b = threadIdx.x;
    const double y = (double)b / 255.0;
    const double n = (double)hist[b];
    double tot[2 * kMaxC + 2];
#pragma unroll
    for (int i = 0; i < 2 * kMaxC + 2; ++i) tot[i] = 0.0;
    tot[0] = n;
    tot[1] = n > 0.0 ? 1.0 : 0.0;
    block_sum_vec<2 * kMaxC + 2>(tot, sh1);
    const double Ntot = tot[0], occ = tot[1];
    if (Ntot <= 0.0 || occ < (double)C) {
        if (threadIdx.x < C) c0[threadIdx.x] = (float)((double)threadIdx.x / (double)(C - 1));
        return;
    }
    const double invN = 1.0 / Ntot;
#pragma unroll
    for (int j = 0; j < C; ++j) {
        mu[j] = ((double)j + 0.5) / (double)C;
        s2[j] = 1.0 / (4.0 * (double)C * (double)C);
        w[j] = 1.0 / (double)C;
    }
    const double two_pi = 6.283185307179586476925286766559;
    for (int it = 0; it < max_iter; ++it) {
        // E step: responsibilities of this bin (R15)
        double r[C];
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const double d = y - mu[j];
            r[j] = w[j] * exp(-d * d / (2.0 * s2[j])) / sqrt(two_pi * s2[j]);
            sum += r[j];
        }
        if (!(sum > 0.0)) {
            int jb = 0;
#pragma unroll
            for (int j = 1; j < C; ++j)
                if (fabs(y - mu[j]) < fabs(y - mu[jb])) jb = j;
#pragma unroll
            for (int j = 0; j < C; ++j) r[j] = (j == jb) ? 1.0 : 0.0;
            sum = 1.0;
        }
        const double isum = 1.0 / sum;
        double v1[2 * kMaxC + 2];
#pragma unroll
        for (int i = 0; i < 2 * kMaxC + 2; ++i) v1[i] = 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const double rr = (n > 0.0) ? r[j] * isum : 0.0;
            r[j] = rr;
            v1[j] = n * rr;              // N_j
            v1[kMaxC + j] = n * rr * y;  // sum y
        }
        block_sum_vec<2 * kMaxC + 2>(v1, sh1);
        double newmu[C], iN[C];
#pragma unroll
        for (int j = 0; j < C; ++j) {
            iN[j] = v1[j] > 1e-12 ? 1.0 / v1[j] : 0.0;
            newmu[j] = (v1[j] > 1e-12) ? v1[kMaxC + j] * iN[j] : mu[j];
        }
        double v2[kMaxC];
#pragma unroll
        for (int j = 0; j < kMaxC; ++j) v2[j] = 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const double d = y - newmu[j];
            v2[j] = n * r[j] * d * d;
        }
        block_sum_vec<kMaxC>(v2, sh2);
        // M step (every thread holds the same sums, so every thread updates)
        double shift = 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            if (v1[j] > 1e-12) {
                w[j] = v1[j] * invN;
                s2[j] = fmax(v2[j] * iN[j], 1e-6);
            }
            shift = fmax(shift, fabs(newmu[j] - mu[j]));
            mu[j] = newmu[j];
        }
        if (shift < 1e-9) break;
    }
    if (threadIdx.x == 0) {
        double m[C];
#pragma unroll
        for (int j = 0; j < C; ++j) m[j] = mu[j];
        for (int i = 1; i < C; ++i) {
            const double t = m[i];
            int k = i - 1;
            while (k >= 0 && m[k] > t) { m[k + 1] = m[k]; --k; }
            m[k + 1] = t;
        }
        bool degen = false;
        for (int j = 1; j < C; ++j)
            if (m[j] - m[j - 1] < 1e-6) degen = true;
        for (int j = 0; j < kMaxC; ++j)
            c0[j] = (j < C) ? (float)(degen ? (double)j / (double)(C - 1) : m[j]) : 0.f;
    }
}

cudaError_t launch_gmm(const int64_t *hist, int C, int max_iter, float *c0, cudaStream_t st) {
    switch (C) {
        case 2: k_gmm<2><<<1, 256, 0, st>>>(hist, max_iter, c0); break;
        case 3: k_gmm<3><<<1, 256, 0, st>>>(hist, max_iter, c0); break;
        case 4: k_gmm<4><<<1, 256, 0, st>>>(hist, max_iter, c0); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- incS
// incS (R26) on a phantom with known truth: cluster j maps to
// the class of its centre's rank (ascending, ties to the lower index); count
// of voxels whose mapped label differs from the truth (integer, exact).
__global__ void k_incs(const uint8_t *labels, const uint8_t *truth, long long n, int C, const float *centers,
                       unsigned long long *count) {
    __shared__ int rank[kMaxC];
    if (threadIdx.x < C) {
        const int j = threadIdx.x;
        int r = 0;
        for (int k = 0; k < C; ++k)
            if (centers[k] < centers[j] || (centers[k] == centers[j] && k < j)) ++r;
        rank[j] = r;
    }
    __syncthreads();
    unsigned long long bad = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int l = labels[i];
        bad += (l >= C || rank[l] != (int)truth[i]) ? 1ull : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}
cudaError_t launch_incs(const uint8_t *labels, const uint8_t *truth, long long n, int C, const float *centers,
                        int64_t *count, cudaStream_t st) {
    if (cudaMemsetAsync(count, 0, sizeof(int64_t), st) != cudaSuccess) return cudaGetLastError();
    long long b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    if (b < 1) b = 1;
    k_incs<<<(int)b, 256, 0, st>>>(labels, truth, n, C, centers, reinterpret_cast<unsigned long long *>(count));
    return cudaGetLastError();
}

// ---------------------------------------------------------------- argmax
// Defuzzification (R13): strict > in cluster order, so ties go
// to the lowest index.
__global__ void k_argmax(const float4 *U, long long n, int C, uint8_t *labels) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 u = U[i];
        const float v[4] = {u.x, u.y, u.z, u.w};
        int best = 0;
        for (int j = 1; j < C; ++j)
            if (v[j] > v[best]) best = j;
        labels[i] = (uint8_t)best;
    }
}
cudaError_t launch_argmax(const float4 *U, long long n, int C, uint8_t *labels, cudaStream_t st) {
    long long b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    k_argmax<<<(int)b, 256, 0, st>>>(U, n, C, labels);
    return cudaGetLastError();
}

}  // namespace pifcm
