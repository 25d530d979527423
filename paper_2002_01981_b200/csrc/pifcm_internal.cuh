// pifcm_internal.cuh -- internal declarations of libpifcm.so (B200, sm_100a).
// Not part of the ABI (see include/pifcm.h).  No code is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pifcm.h"

namespace pifcm {

// ---------------------------------------------------------------- constants
constexpr int kMaxC = 4;          // AoS-C4 rows: one float4 per voxel
constexpr int kNR = 2 * kMaxC + 2; // partial record: num[4], den[4], J, max|du|
constexpr int kMaxV = 3;          // shells on the device path (Eq. 9-10; v = 1 the hot kernel, 2..3 step_shells.cu)
constexpr float kAFloor = 1e-9f;  // R4: floor of 1 - lam H - xi F (Eq. 4)
constexpr double kDenEps = 1e-12; // R9: keep c_j if sum u^m < 1e-12 (Eq. 3)
// Ill-conditioned voxels: u_j moves by u_j (1 - u_j) / ((m-1) a_j) per unit
// relative change of the Eq. 4 factor a_j.  The fp32 factors are accurate to
// kAErr (absolute; sums of <= 26 positive fp32 terms, a ratio and two FMAs),
// so a voxel whose sensitivity K = sum_j u_j (1 - u_j) / ((m-1) a_j) exceeds
// kKMax = kUTol / kAErr is re-evaluated from the definitions in fp64
// (DESIGN.md §Numerics).  kUTol leaves a 4x margin to the 1e-4 tolerance.
#ifndef PIFCM_KMAX
#define PIFCM_KMAX 25.0f
#endif
constexpr float kAErr = 1e-6f;
constexpr float kUTol = 2.5e-5f;
constexpr float kKMax = PIFCM_KMAX;  // = kUTol / kAErr

// Stencil step tiling (one CTA = TX x TY voxels per plane, marching TZ planes).
constexpr int kTX = 32;             // one warp along x: 512 B coalesced rows
#ifndef PIFCM_WARPS_Y
#define PIFCM_WARPS_Y 4
#endif
#ifndef PIFCM_RY
#define PIFCM_RY 4
#endif
constexpr int kWarpsY = PIFCM_WARPS_Y;  // warps per CTA, stacked in y
constexpr int kRY = PIFCM_RY;           // consecutive y rows per thread (register blocking)
constexpr int kTY = kWarpsY * kRY;  // 16
constexpr int kSX = kTX + 2;        // haloed smem row length
constexpr int kSY = kTY + 2;        // haloed smem rows
#ifndef PIFCM_TZ
#define PIFCM_TZ 32
#endif
constexpr int kTZ = PIFCM_TZ;       // planes per CTA (z-chunk) for deep grids
constexpr int kTZMin = 8;           // smallest z-chunk used to fill a wave
constexpr int kStepThreads = kTX * kWarpsY;
#ifndef PIFCM_TYB2D
#define PIFCM_TYB2D 4
#endif
constexpr int kTYB2D = PIFCM_TYB2D;  // 2D step: tiles per CTA (a column in y)

// Pointwise (FCM, lambda = xi = 0) step.
constexpr int kPwThreads = 256;
constexpr int kPwSpan = 8;  // voxels per lane per span

// ------------------------------------------------------------ step arguments
struct StepArgs {
    const float *x;      // [nz][ny][pitch]
    int nx, ny, nz, pitch;  // nz = planes in the arrays (slab mode: local planes + 2 halos)
    long long nvox;      // nx*ny*nz  (float4 rows per state)
    int z_lo, nz_t;      // target planes [z_lo, z_lo + nz_t) in array coordinates
    int goff, nz_g;      // global z of array plane 0; planes of the whole volume
    int canonical;       // whole volume with the fixed global 16-plane chunks of the slab mode
    const float4 *U_in;  // base of input states
    float4 *U_out;       // base of output states
    const int *in_idx;   // nullable: state p reads U_in + in_idx[p]*nvox (else p*nvox)
    const int *out_idx;  // nullable: state p writes U_out + out_idx[p]*nvox
    float *centers;      // [P][4] (read at kernel start)
    const double *lam_xi;// [P][2]  (already offset to this process's first particle)
    double *partials;    // [P][nblk][kNR]
    int nblk;            // partial records per state
    const double *stats; // nullable: skip state p if stats[4p+3] != 0 (converged)
    const int *stop;     // nullable: skip everything if *stop != 0
    int tiles_x, tiles_y, zchunks, tz;  // tz = planes per z-chunk
    float m, inv_m1;     // m, 1/(m-1)
    int q_mode;
    int first;           // FCM first iteration: U_in not read, max|du| := 1
    int n_in_states;     // states addressable from U_in (TMA tensor-map extent)
    int want_du;         // accumulate max|u_new - u_old| (convergence tests)
    // fused finalisation (Eq. 3 / Eq. 1) by the last CTA of each state
    unsigned *counters;  // [P] arrival counters, 0 between launches
    int C;
    double *fitness;     // nullable [P]
    double *stats_out;   // nullable [P][4] {J, du, iters, converged} (same array as stats)
    float eps;
    int *status;         // nullable: PIFCM_ENUMERIC on a non-finite J
    float4 *hf;          // non-null: emit H (float4) and F (float4) per voxel [nvox][2] instead of a step
    int v;               // neighbourhood shells (Eq. 9-10): 1 = the 26-neighbourhood, 2 = two shells
    float wsh[kMaxV];    // Eq. 10 shell weights W_1 .. W_v (v >= 2)
    double wshd[kMaxV];  // the same in fp64 (ill-conditioned re-evaluation)
};

// Swarm state in the workspace (all device pointers).
struct SwarmDev {
    int *hdr;        // [16] ints: see kH* below
    double *dhdr;    // [16] doubles: see kD* below
    double *pos;     // [P][2] current positions (lambda, xi)
    double *vel;     // [P][2]
    double *pbf;     // [P] pbest fitness
    double *pbx;     // [P][2] pbest positions
    double *fit;     // [P] fitness of the current generation
    double *evalpos; // [P][2] positions the current generation was evaluated at
    int *cur;        // [Pl] slot holding each local particle's state
    int *nxt;        // [Pl] slot the next evaluation writes
    float *gbest_c;  // [4]
    float *centers;  // [Pl][4]
};
// header int indices
constexpr int kHGen = 0, kHGbest = 1, kHGbestSlot = 2, kHImproved = 3, kHCalm = 4,
              kHStop = 5, kHStatus = 6, kHInit = 7, kHNotImproved = 8, kHHfValid = 9;
// header double indices
constexpr int kDPrevGf = 0, kDGbestJ = 1, kDGbestL = 2, kDGbestX = 3;

struct PsoUpdateArgs {
    SwarmDev s;
    int P, Pl, p0, ring_k, patience, nslots;
    int mode;  // pifcm_fitness: CHAINED / ANCHORED / LEADER
    int batched;  // CHAINED with batched evaluation: next slots assigned per batch (k_assign_batch)
    double tol, vmax;
    uint32_t key0, key1;
    // optional per-generation record (pifcm_pso_trace): f[t][P], evaluation
    // positions [t][P][2], gbest index [t] for t < tr_max; NULL = off
    double *tr_f, *tr_pos;
    int *tr_gbest;
    int tr_max;
};

// z-slab exchange over peer memory (p2p.cu)
constexpr int kMaxPeers = 16;
struct P2PPut {
    const float4 *src;           // this rank's new states [P][nz+2H][ny][nx]
    long long plane, state;      // voxels per plane, per state (incl. halos)
    int nz, P, H;                // local planes, states, halo planes per side (= v)
    float4 *lo_dst;              // rank-1's buffer + its upper halo planes (nullable)
    long long lo_state;          // rank-1's voxels per state
    float4 *hi_dst;              // rank+1's buffer + its lower halo planes (nullable)
    long long hi_state;
    const double *rec_src;       // this rank's records [P][nrec][kNR] (nullable)
    int nrec, nrec_max, world, rank;
    double *rec_dst[kMaxPeers];  // every rank's gathered buffer [world][P][nrec_max][kNR]
    unsigned *flags[kMaxPeers];  // every rank's flags [world]
    unsigned *counter;           // this rank's block-arrival counter (0 between launches)
    unsigned epoch;
};

// x of a quantised value v for the volume range [lo, hi] (Alg. 2 step 1,
// PAPER:173-174; R16: a constant volume maps to 0): the integer difference
// and one correctly rounded fp32 division.  k_normalize and the
// value-histogram FCM (fcm_hist.cu) both use it, so they see the same x.
__device__ __forceinline__ float normalize_q(int v, int lo, int hi) {
    return hi > lo ? __fdiv_rn((float)(v - lo), (float)(hi - lo)) : 0.f;
}

// The FCM start on the value histogram (fcm_hist.cu).
struct FcmHistArgs {
    const int64_t *counts;  // [nvals] voxels per raw value (u8: 256, u16: 65536)
    int nvals;
    const unsigned *mm;     // {min, max} raw values of the volume
    const float *c0;        // [4] start centres
    int max_iter;
    float eps, m, inv_m1;
    float *xs;              // scratch [nvals]: x of the occupied values
    double *ns;             // scratch [nvals]: their counts
    float4 *up;             // scratch [nvals]: their rows of the previous iteration
    float *c_prev;          // [4] out: the centres the last iteration's rows used
    float *c_out;           // [4] out: the centres after the last iteration (Eq. 3)
    double *stats;          // [4] out: {J, max|du|, iterations, converged}
    int *status;            // nullable: PIFCM_ENUMERIC on a non-finite J
};

// ---------------------------------------------------------------- launchers
// All return cudaGetLastError() of the launch.
cudaError_t launch_step(const StepArgs &a, int C, bool stencil, int P, cudaStream_t st);
cudaError_t launch_step_shells(const StepArgs &a, int C, int P, cudaStream_t st);
// the iterations of one 2D state in one cooperative launch; *used = false when
// its CTAs cannot all be resident (step.cu)
cudaError_t launch_2d_loop(const StepArgs &a, int C, float4 *UA, float4 *UB, int iters, unsigned *gbar,
                           cudaStream_t st, bool *used);  // step_shells.cu (v = 2, 3)
int step_nblk(int nx, int ny, int nz, bool stencil, int P);
int slab_tz(int nx, int ny, int nz_total);
int step_nblk_max(int nx, int ny, int nz);
int step_zchunks(int nx, int ny, int nz, int P);
cudaError_t launch_fixup_copy(const float4 *scratch, float4 *out, long long nvox, int P,
                              const double *stats, int iters, cudaStream_t st);
cudaError_t launch_pso_init(SwarmDev s, int P, int Pl, int p0, double v0, uint32_t k0,
                            uint32_t k1, const float *c0, int nslots, cudaStream_t st);
cudaError_t launch_pso_update(const PsoUpdateArgs &a, cudaStream_t st);
cudaError_t launch_assign_batch(SwarmDev s, int Pl, int b0, int nb, int nslots, cudaStream_t st);
cudaError_t launch_minmax(const void *vol, int dtype, long long n, unsigned int *mm, cudaStream_t st);
cudaError_t launch_normalize(const void *vol, int dtype, int nx, int ny, int nz, int pitch,
                             const unsigned int *mm, float *x, cudaStream_t st);
cudaError_t launch_hist(const void *vol, int dtype, long long n, const unsigned int *mm, int64_t *hist,
                        cudaStream_t st);
cudaError_t launch_minmax_u8(const uint8_t *vol, long long n, unsigned int *mm, cudaStream_t st);
cudaError_t launch_normalize_u8(const uint8_t *vol, int nx, int ny, int nz, int pitch,
                                const unsigned int *mm, float *x, cudaStream_t st);
cudaError_t launch_hist_u8(const uint8_t *vol, long long n, const unsigned int *mm,
                           int64_t *hist, cudaStream_t st);
cudaError_t launch_value_hist(const void *vol, int dtype, long long n, int64_t *counts, cudaStream_t st);
cudaError_t launch_fcm_hist(const FcmHistArgs &a, int C, bool m2, cudaStream_t st);
cudaError_t launch_fcm_memberships(const float *x, int nx, int ny, int nz, int pitch, const float *c, int C,
                                   float m, float4 *U, cudaStream_t st);
size_t small2d_smem(int nx, int ny);
cudaError_t launch_iterate_small2d(const float *x, int nx, int ny, int pitch, const float4 *U_in, float4 *U_out,
                                   float *centers, const double *lam_xi, int P, int iters, float eps, float m,
                                   int q_mode, int C, double *stats, int *status, cudaStream_t st);
cudaError_t launch_gmm(const int64_t *hist, int C, int max_iter, float *c0, cudaStream_t st);
cudaError_t launch_incs(const uint8_t *labels, const uint8_t *truth, long long n, int C, const float *centers,
                        int64_t *count, cudaStream_t st);
cudaError_t launch_argmax(const float4 *U, long long n, int C, uint8_t *labels,
                          cudaStream_t st);
cudaError_t launch_gather_gbest(const float4 *slots, long long nvox, const int *hdr,
                                const float *gbest_c, float4 *U_out, float *c_out,
                                cudaStream_t st);
// fitness modes ANCHORED / LEADER (fitness.cu)
cudaError_t launch_eval_shared(const float *x, int nx, int ny, int nz, int pitch, const float4 *hf,
                               const float *centers, const double *pos, int P, int C, float m, double *partials,
                               int *nparts, cudaStream_t st);
int eval_shared_parts(long long nvox, int P);
cudaError_t launch_fit_sum(const double *partials, int nparts, int P, double *fitness, int *status,
                           cudaStream_t st);
cudaError_t launch_mode_pre(SwarmDev s, const float *shared_c, double *lamxi, int mode, cudaStream_t st);
cudaError_t launch_leader_post(SwarmDev s, const float *shared_c, cudaStream_t st);
cudaError_t launch_set_hdr(int *hdr, int idx, int value, cudaStream_t st);
cudaError_t launch_p2p_put(const P2PPut &a, cudaStream_t st);
cudaError_t launch_p2p_wait(const unsigned *flags, int world, unsigned epoch, int *status, cudaStream_t st);
cudaError_t launch_set_lamxi(double *dst, const double *dhdr, cudaStream_t st);
cudaError_t launch_slab_finalize(int C, int P, int world, int nrec, const int *counts, const double *records,
                                 float *centers, double *stats, double *fitness, float eps, int *status,
                                 cudaStream_t st);
cudaError_t launch_halo_copy(const float4 *src, long long src_state, float4 *dst, long long dst_state,
                             long long plane, int P, bool zero, cudaStream_t st, const int *src_idx = nullptr,
                             const int *dst_idx = nullptr);

}  // namespace pifcm
