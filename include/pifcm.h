/*
 * pifcm.h -- C ABI of libpifcm.so, the B200 (sm_100a) hot path of 3DPIFCM
 * (Agranonik, Herman, Last, "Parallel 3DPIFCM Algorithm for Noisy Brain MRI
 * Images", arXiv 2002.01981).
 *
 * Citation shorthand: PAPER:N = line N of the paper text, with the
 * equation / algorithm it falls in.  "Rk" names a reading of an ambiguous
 * passage, listed in DESIGN.md §Readings.
 *
 * What the library computes ("the step function"):
 *   one IFCM iteration per voxel i and cluster j, from the previous
 *   memberships U (Jacobi, R7):
 *     g_ik  = |x_i - x_k|                               Eq. 6
 *     q_ik  = dX^2 + dY^2 + dZ^2, q2 per R1            Eq. 8
 *     k in NB_i = 26-neighbourhood (v = 1)             Eq. 9, R2
 *     H_ij  = sum_k u_kj g_ik / sum_k g_ik  (0 if 0/0) Eq. 5, R3
 *     F_ij  = sum_k u_kj^2 q2_ik / sum_k q2_ik          Eq. 7
 *     d2_ij = (x_i - c_j)^2 max(1 - lam H_ij - xi F_ij, 1e-9)   Eq. 4, R4
 *     u_ij  = 1 / sum_k (d2_ij / d2_ik)^{1/(m-1)}      Eq. 2, R5
 *     c_j   = sum_i u_ij^m x_i / sum_i u_ij^m          Eq. 3, R9
 *     J     = sum_i sum_j u_ij^m d2_ij                 Eq. 1, R8
 *   evaluated for every PSO particle's (lam, xi) (Alg. 1 steps 4-8,
 *   PAPER:98-102), inside the whole pipeline of Alg. 1 / Alg. 2
 *   (PAPER:91-106, 171-187).
 *
 * Conventions for every call:
 *   - Ownership: every buffer is borrowed from the caller (device memory from
 *     torch / cudaMalloc, or host memory where stated).  The library owns only
 *     the opaque context (streams/events/host scratch).  Device scratch is the
 *     caller's workspace `ws`, sized by pifcm_workspace_size(); the library
 *     never calls cudaMalloc on the compute path.
 *   - Errors: a negative pifcm_status; no exception crosses the ABI.  All
 *     arguments are validated before any launch; on failure nothing is
 *     launched and pifcm_last_error() describes the problem.  Asynchronous
 *     CUDA errors surface at the next synchronous call as PIFCM_ECUDA.
 *   - Asynchrony: calls marked "async" enqueue on `stream` and return; calls
 *     marked "sync" synchronise `stream` before returning.
 *   - Determinism: every reduction sums fixed-size per-block fp64 partials in
 *     a fixed order, so results are bit-identical run to run.
 *   - A context is single-threaded.
 *
 * Device layouts:
 *   x        fp32 [nz][ny][pitch], pitch >= nx, pitch % 4 == 0 (16-byte rows);
 *            normalised intensities in [0,1] (Alg. 2 step 1).
 *   U        fp32 "AoS-C4" [P][nz][ny][nx][4]: one 16-byte row per voxel,
 *            u_i0..u_i(C-1) then zeros.  Rows must sum to 1 (they do for any
 *            U the library writes).
 *   centers  fp32 [P][4] (c_0..c_{C-1}, rest ignored).
 *   lam_xi   fp64 [P][2] (lambda, xi) in [0,1]^2.
 *   labels   u8 [nz][ny][nx].
 */
#ifndef PIFCM_H
#define PIFCM_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is exported even under -fvisibility=hidden */
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *pifcm_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    PIFCM_OK = 0,
    PIFCM_EINVAL = -1,   /* invalid argument (range, null pointer, C > 4 ...) */
    PIFCM_EALIGN = -2,   /* pitch / pointer alignment violated (16-byte rows required) */
    PIFCM_ENOMEM = -3,   /* workspace smaller than pifcm_workspace_size() */
    PIFCM_ECUDA = -4,    /* a CUDA runtime error (launch or asynchronous) */
    PIFCM_ENCCL = -5,    /* the context's communicator failed (NCCL load / init / collective, or a host collective) */
    PIFCM_ENUMERIC = -6, /* non-finite cost J */
    PIFCM_ESTATE = -7    /* call order violated (e.g. pso_step before pso_init) */
} pifcm_status;

typedef enum { PIFCM_Q_LITERAL = 0, PIFCM_Q_SQEUCLID = 1 } pifcm_qmode; /* R1 */
/* Fitness of a PSO particle (R11): CHAINED = each particle owns a
 * state and advances it one step per generation; ANCHORED = every evaluation
 * is one step from the shared start (U0, c0); LEADER = every evaluation is one
 * step from a shared state that follows the gbest's evaluation (R22).  In
 * ANCHORED / LEADER the particle-invariant H, F of the shared state are
 * computed once per state and the P fitness values are pointwise. */
typedef enum { PIFCM_FIT_CHAINED = 0, PIFCM_FIT_ANCHORED = 1, PIFCM_FIT_LEADER = 2 } pifcm_fitness;
typedef enum { PIFCM_U8 = 0, PIFCM_U16 = 1, PIFCM_F32 = 2 } pifcm_dtype;

typedef struct pifcm_ctx pifcm_ctx;

/* Volume extent.  Alg. 1 input "img3d - a 3D matrix of pixel intensities"
 * (PAPER:93).  nz == 1 is the 2D case (8-neighbourhood).
 * z-slab mode (nz_total > 0, only for the pifcm_slab_* calls): this process
 * holds the planes [z0, z0 + nz) of a volume of nz_total planes; its x and U
 * arrays then have nz + 2v planes for the neighbourhood radius v of the
 * pifcm_ifcm_cfg (Eq. 9-10), plane 0 being global z0 - v and plane
 * nz + 2v - 1 global z0 + nz + v - 1 (v halo planes per side; v = 1: nz + 2
 * planes, halos at 0 and nz + 1).  With tz = pifcm_slab_chunk(nx, ny,
 * nz_total), z0 must be a multiple of tz and every slab but the last must
 * have a multiple of tz planes (the slab reductions use global chunks of tz
 * planes, which makes them independent of the number of slabs).
 * nz_total = 0 (or z0 = 0, nz_total = nz): whole volume. */
typedef struct {
    int32_t nx, ny, nz;
    int32_t pitch;    /* elements per x row of the intensity volume; >= nx, % 4 == 0 */
    int32_t z0;       /* z-slab: first global plane held (0 otherwise)                 */
    int32_t nz_total; /* z-slab: planes of the whole volume (0: not a slab)             */
} pifcm_grid;

/* Method parameters.  Alg. 1 inputs c, v, h, m, epsilon. */
typedef struct {
    int32_t C;        /* clusters, 2..4 on the device path                      */
    float m;          /* fuzzifier, m > 1 (Eq. 2); m == 2 takes a fast path     */
    int32_t v;        /* shells (Eq. 9-10, R2): 1 (26 neighbours), 2 (124), 3 (342) */
    float h;          /* Eq. 10 decay (> 0); irrelevant at v == 1               */
    int32_t q_mode;   /* pifcm_qmode (R1)                                       */
    float eps;        /* stop when max|u_new - u_old| < eps (R14); <= 0: never   */
    int32_t max_iter; /* iteration cap of the FCM start and final IFCM (R14)    */
} pifcm_ifcm_cfg;

/* PSO parameters (Alg. 1 steps 3-9; R12). */
typedef struct {
    int32_t P;          /* particles, 1..1024                                     */
    int32_t ring_k;     /* lbest ring radius (>= 0)                               */
    int32_t max_gen;    /* generation cap (>= 1)                                  */
    int32_t patience;   /* stop after `patience` calm generations; <= 0: never    */
    double tol;         /* calm: relative decrease of the gbest J < tol           */
    double v0;          /* initial |velocity| bound                               */
    double vmax;        /* velocity clamp                                         */
    uint64_t seed;      /* Philox4x32-10 key                                      */
    int32_t fitness_mode; /* pifcm_fitness (ANCHORED / LEADER: P <= 128)           */
    int32_t p_begin;    /* this process evaluates particles [p_begin, p_end)      */
    int32_t p_end;      /*   (particle sharding; 0,0 means all P)                 */
    int32_t eval_batch; /* CHAINED: evaluate this process's particles in launches of
                           eval_batch states, reusing the slots the previous batch
                           released: Pl + eval_batch + 1 state slots instead of
                           2 Pl + 1 (0 or >= Pl: one launch).  Results are
                           bit-identical for any value.                           */
} pifcm_pso_cfg;

/* Host-side summary of a PSO run (Alg. 1 step 10). */
typedef struct {
    double lambda, xi, J;     /* gbest position and fitness                       */
    int32_t generations;      /* generations run                                  */
    int32_t gbest_particle;   /* global particle index of the gbest               */
    float centers[4];         /* gbest centres (the state its evaluation produced)*/
} pifcm_pso_result;

/* Host-side summary of a whole segmentation. */
typedef struct {
    pifcm_pso_result pso;
    int32_t fcm_iters;        /* iterations of the FCM start (Alg. 1 step 2)      */
    int32_t final_iters;      /* iterations of the final IFCM (Alg. 1 step 11)    */
    float c_init[4];          /* GMM centres (R15)                                */
    float centers[4];         /* final centres                                    */
    double t_norm, t_init, t_pso, t_final, t_total; /* seconds (CUDA events)      */
} pifcm_report;

/* ---------------------------------------------------------------- context */
/* Create a context bound to CUDA device `device`.  Returns PIFCM_OK or
 * PIFCM_ECUDA / PIFCM_EINVAL.  *out receives the context. */
int pifcm_ctx_create(int device, pifcm_ctx **out);
void pifcm_ctx_destroy(pifcm_ctx *ctx);
/* Message describing the last non-OK status returned with this ctx (never NULL). */
const char *pifcm_last_error(const pifcm_ctx *ctx);
/* Library version string. */
const char *pifcm_version(void);

/* ----------------------------------------------------------- multi-process */
/* The particle-sharded pipeline (SURVEY 8(b) pifcm_dist, 8(e)).  The PSO's
 * particles are independent within a generation (Alg. 1 step 4), so
 * rank r of `world` evaluates the contiguous range pifcm_dist_range(P, world,
 * r) (20 over 8 -> 3,3,3,3,2,2,2,2); the only exchanges are the all-gather of
 * the fitness vector every generation (step 4 -> 5) and the broadcast of the
 * gbest state from its owner before the final IFCM (steps 10-11,
 * PAPER:104-105).  Every rank runs the identical fp64 PSO update and the
 * final IFCM in the canonical decomposition, so labels, centres and
 * (lambda*, xi*) are bit-identical to the single-process pifcm_segment on
 * every rank. */
typedef struct {
    int32_t rank, world;             /* this process, number of processes        */
    const uint8_t *nccl_unique_id;   /* 128 bytes from pifcm_nccl_unique_id (one
                                        rank creates it, the caller shares it);
                                        ignored when host collectives are given */
    int32_t shard;                   /* 0 = particles (the only C-level sharding;
                                        the z-slab final IFCM is pifcm_slab_*)   */
} pifcm_dist;
/* Host-memory collectives supplied by the caller (gloo, MPI, ...; e.g. ranks
 * sharing one GPU, which NCCL refuses).  Both return 0 on success; they are
 * called synchronously, in the same order, on every rank. */
typedef struct {
    void *user;
    /* dst[world][bytes] <- every rank's src[bytes], in rank order */
    int (*allgather)(void *user, const void *src, void *dst, size_t bytes);
    /* buf[bytes] on every rank <- buf of rank `root` */
    int (*broadcast)(void *user, void *buf, size_t bytes, int32_t root);
} pifcm_host_coll;
/* 128-byte NCCL unique id (ncclGetUniqueId of the libnccl.so.2 the library
 * loads with dlopen).  PIFCM_ENCCL when NCCL cannot be loaded. */
int pifcm_nccl_unique_id(uint8_t id[128]);
/* Attach a communicator to ctx (the ctx owns it; a previous one is freed):
 * NCCL (ncclCommInitRank on ctx's device; collective over all ranks, blocks
 * until every rank has called it) unless `coll` is non-NULL, in which case
 * the caller's host collectives are used.  world == 1 detaches.  Errors:
 * PIFCM_EINVAL (rank outside [0, world), shard != 0, missing id / callbacks),
 * PIFCM_ENCCL (NCCL load or init). */
int pifcm_ctx_dist(pifcm_ctx *ctx, const pifcm_dist *dist, const pifcm_host_coll *coll);
/* The particle range [*p_begin, *p_end) of `rank`: what pifcm_pso_cfg.p_begin
 * / p_end must hold (and the workspace be sized for) on that rank. */
int pifcm_dist_range(int32_t P, int32_t world, int32_t rank, int32_t *p_begin, int32_t *p_end);

/* --------------------------------------------------------------- workspace */
/* Bytes of device workspace needed by pso_* / segment calls for this grid and
 * configuration (pso may be NULL for pifcm_iterate-only use, in which case the
 * size covers pifcm_iterate with P = 1).  PIFCM_EINVAL on invalid arguments. */
int pifcm_workspace_size(const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                         const pifcm_pso_cfg *pso, size_t *bytes);
/* Bytes of device scratch pifcm_iterate needs for P states and `iters`
 * iterations (0 when iters == 1). */
int pifcm_iterate_workspace_size(const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                                 int32_t P, int32_t iters, size_t *bytes);

/* ------------------------------------------------------------------ iterate */
/* `iters` Jacobi IFCM iterations (Alg. 2 steps 6-8,
 * PAPER:179-181) for P independent states over one shared volume: state p
 * uses (lam_xi[p], centers[p], U_in[p]).  Async.
 *   x        dev fp32 [nz][ny][pitch]
 *   U_in     dev fp32 [P][nz][ny][nx][4]   (read only)
 *   U_out    dev fp32 [P][nz][ny][nx][4]   (result; must not alias U_in)
 *   centers  dev fp32 [P][4]   in: c used by the first iteration; out: Eq. 3
 *   lam_xi   dev fp64 [P][2]   lambda, xi in [0,1] (lambda = xi = 0: plain FCM)
 *   stats    dev fp64 [P][4]   out, nullable: {J, max|du|, iterations, converged}
 *            of the last iteration run for that state.  J follows R8.
 *   ws       dev scratch of pifcm_iterate_workspace_size() bytes (NULL if 0).
 * With cfg->eps > 0 a state stops once its max|du| < eps (its U_out then
 * holds the converged U); otherwise exactly `iters` iterations run.
 * A 2D image of at most 4096 voxels (e.g. the 32 x 32 config C1) runs all
 * iterations in one launch, one CTA per state holding the image in shared
 * memory; any other grid runs one launch per iteration.
 * Errors: PIFCM_EINVAL (dims, C, m, P < 1, iters < 1, lam/xi range is not
 * checked on device data), PIFCM_EALIGN (pitch), PIFCM_ENOMEM (ws too small),
 * PIFCM_ECUDA. */
int pifcm_iterate(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                  const float *x, const float *U_in, float *U_out, float *centers,
                  const double *lam_xi, int32_t P, int32_t iters, double *stats,
                  void *ws, size_t ws_bytes, pifcm_stream stream);

/* pifcm_iterate with flags: PIFCM_ITER_CANONICAL runs the neighbourhood
 * launches in the canonical z-chunk decomposition (pifcm_slab_chunk), the one
 * pifcm_segment's final IFCM and every z-slab split use, so the results are
 * bit-identical to those (used by multi-rank pipelines that run the final
 * IFCM replicated on every rank). */
#define PIFCM_ITER_CANONICAL 1
/* With PIFCM_ITER_CANONICAL, a 2D image (nz = 1, v = 1), P = 1 and iters > 1
 * run every iteration in one cooperative launch (a grid barrier and the
 * canonical finalisation between the steps; results bit-identical to one
 * launch per step) when its CTAs can all be resident; PIFCM_ITER_PER_STEP
 * forces one launch per iteration. */
#define PIFCM_ITER_PER_STEP 2
int pifcm_iterate_ex(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                     const float *x, const float *U_in, float *U_out, float *centers,
                     const double *lam_xi, int32_t P, int32_t iters, double *stats,
                     void *ws, size_t ws_bytes, int32_t flags, pifcm_stream stream);

/* --------------------------------------------------------------------- PSO */
/* Initialise the swarm (Alg. 1 step 3; Alg. 2 step 3)
 * in the workspace: positions ~ U[0,1]^2 and velocities ~ U[-v0,v0]^2 from
 * Philox (R12), every particle's state := (U0, c0).  Async.
 *   U0 dev fp32 [nz][ny][nx][4]; c0 dev fp32 [4].
 * Errors: PIFCM_EINVAL, PIFCM_ENOMEM, PIFCM_ECUDA. */
int pifcm_pso_init(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                   const pifcm_pso_cfg *pso, const float *U0, const float *c0,
                   void *ws, size_t ws_bytes, pifcm_stream stream);

/* Fitness evaluation of this process's particles [p_begin, p_end) for the
 * current generation (Alg. 1 step 4; fitness modes R11 / R22): the
 * J of one IFCM step of the particle's state (CHAINED) or of the shared state
 * (ANCHORED, LEADER) at its (lambda, xi); the J values land in the fitness
 * vector returned by pifcm_pso_fitness_ptr().  x must stay the same during a
 * PSO run (ANCHORED computes the shared H, F once).  Async. */
int pifcm_pso_eval(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                   const pifcm_pso_cfg *pso, const float *x, void *ws, size_t ws_bytes,
                   pifcm_stream stream);

/* Device pointer to the fitness vector fp64 [P] inside `ws` (so that a
 * multi-process caller can all-gather it between eval and update).  Entries
 * outside [p_begin, p_end) must be filled by the caller before update. */
int pifcm_pso_fitness_ptr(const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                          const pifcm_pso_cfg *pso, void *ws, double **fitness);

/* PSO bookkeeping and move after all P fitnesses are known (Alg. 1 steps 5-8,
 * PAPER:99-102): pbest (strict <), ring lbest, velocity, fly, gbest snapshot
 * and the stop test of step 9 (R12).  Identical on every process.  ANCHORED:
 * on an improvement the snapshot step from the start runs here; LEADER: the
 * shared state advances here by the gbest's step (x dev fp32 [nz][ny][pitch],
 * required for those modes, may be NULL for CHAINED).  Async. */
int pifcm_pso_update(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                     const pifcm_pso_cfg *pso, const float *x, void *ws, size_t ws_bytes,
                     pifcm_stream stream);

/* Per-generation record of the swarm (a test / debugging aid, SURVEY 5
 * tracing): while set, every pifcm_pso_update of this ctx (and so
 * pifcm_pso_step / _run / pifcm_segment) writes, for its generation t <
 * max_gen, the fitness vector it consumed f[t][P] (Alg. 1 step 4), the
 * positions it was evaluated at pos[t][P][2] and the gbest particle after the
 * update gbest[t] (step 8) into these caller-owned device buffers.  The
 * generation counter restarts at pifcm_pso_init.  All three NULL switch it
 * off; a partial set, or max_gen < 1, is PIFCM_EINVAL.  No synchronisation. */
int pifcm_pso_trace(pifcm_ctx *ctx, double *f, double *pos, int32_t *gbest, int32_t max_gen);

/* One generation on one process: pifcm_pso_eval + pifcm_pso_update.  Async. */
int pifcm_pso_step(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                   const pifcm_pso_cfg *pso, const float *x, void *ws, size_t ws_bytes,
                   pifcm_stream stream);

/* Read the swarm summary (sync).  `stopped` (nullable) receives 1 once the
 * step-9 stop rule fired. */
int pifcm_pso_result_get(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                         const pifcm_pso_cfg *pso, void *ws, pifcm_pso_result *out,
                         int32_t *stopped, pifcm_stream stream);

/* Copy the gbest state (the U and centres its evaluation produced, Alg. 1
 * step 10) to U_out [nz][ny][nx][4] / c_out [4] (device).  PIFCM_ESTATE when
 * the gbest particle is not evaluated by this process.  Async. */
int pifcm_pso_gbest_state(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                          const pifcm_pso_cfg *pso, void *ws, float *U_out, float *c_out,
                          pifcm_stream stream);

/* Whole PSO (Alg. 1 steps 3-10): init from (U0, c0), generations until the
 * stop rule or max_gen, summary into *out.  Single process.  Sync. */
int pifcm_pso_run(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                  const pifcm_pso_cfg *pso, const float *x, const float *U0, const float *c0,
                  void *ws, size_t ws_bytes, pifcm_pso_result *out, pifcm_stream stream);

/* ----------------------------------------------------------- pipeline parts */
/* Alg. 2 step 1: global min-max normalisation of a device u8
 * volume [nz][ny][nx] into x [nz][ny][pitch] (constant volume -> 0, R16) and
 * the 256-bin histogram of R15 into hist (dev int64 [256], nullable).  Async. */
int pifcm_normalize_u8(pifcm_ctx *ctx, const pifcm_grid *grid, const uint8_t *vol, float *x,
                       int64_t *hist, void *ws, size_t ws_bytes, pifcm_stream stream);
/* The same for a volume of type dtype (PIFCM_U8, PIFCM_U16 --
 * integer arithmetic as u8 -- or PIFCM_F32: x = (v - min) / (max - min) and
 * the R15 bin floor((v - min) * 255 / (max - min) + 0.5) in fp64, values
 * assumed finite).  PIFCM_EINVAL for another dtype.  Async. */
int pifcm_normalize(pifcm_ctx *ctx, const pifcm_grid *grid, const void *vol, int32_t dtype, float *x,
                    int64_t *hist, void *ws, size_t ws_bytes, pifcm_stream stream);

/* R15 "Modified_FCM with Gaussian mixture model": 1-D EM on
 * the 256-bin histogram -> C initial centres (fp32 [4], device).  Async. */
int pifcm_gmm_init(pifcm_ctx *ctx, int32_t C, const int64_t *hist, float *c0, void *ws,
                   size_t ws_bytes, pifcm_stream stream);

/* The FCM start of a quantised volume on its value histogram (
 * Alg. 1 step 2; Alg. 2 step 5; DESIGN R24).  FCM is the
 * IFCM step at lambda = xi = 0, where Eq. 4's factor is 1 and a voxel's Eq. 2
 * row depends on its x and the centres only, so the Eq. 3 / Eq. 1 sums over
 * voxels are the count-weighted sums over the distinct values.
 *   pifcm_value_hist: counts[v] += number of voxels of raw value v among the
 *     n values at vol (dev; dtype PIFCM_U8 -> 256 entries, PIFCM_U16 -> 65536
 *     entries, dev int64, zeroed by the caller; a z-slab caller sums the
 *     ranks' counts).  PIFCM_EINVAL for PIFCM_F32.  Async.
 *   pifcm_fcm_hist: FCM iterations from the centres c0 (dev fp32 [4]) on the
 *     counts of a volume with raw range mm (dev uint32 {min, max}, as
 *     pifcm_minmax_u8 / pifcm_normalize write it) until max|du| < cfg->eps
 *     (the first iteration never stops, R14) or cfg->max_iter.  Writes c_prev
 *     (dev fp32 [4]: the centres the last iteration's memberships used),
 *     c_out (dev fp32 [4]: Eq. 3 centres after it) and stats (dev fp64 [4]:
 *     {J, max|du|, iterations, converged}).  ws: >= the size
 *     pifcm_fcm_hist_workspace_size gives for dtype (device, 256-B aligned).
 *     Async; a non-finite J sets the status read by the next sync call.
 *   pifcm_fcm_memberships: U (dev fp32 [nz][ny][nx][4]) = the Eq. 2 rows of
 *     x (dev [nz][ny][pitch]) at the centres c (dev [4]) with lambda = xi = 0:
 *     with c = c_prev, the memberships of the FCM start.  Async. */
int pifcm_value_hist(pifcm_ctx *ctx, const void *vol, int32_t dtype, int64_t n, int64_t *counts,
                     pifcm_stream stream);
int pifcm_fcm_hist_workspace_size(int32_t dtype, size_t *bytes);
int pifcm_fcm_hist(pifcm_ctx *ctx, const pifcm_ifcm_cfg *cfg, int32_t dtype, const uint32_t *mm,
                   const int64_t *counts, const float *c0, float *c_prev, float *c_out, double *stats, void *ws,
                   size_t ws_bytes, pifcm_stream stream);
int pifcm_fcm_memberships(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t C, float m, const float *x,
                          const float *c, float *U, pifcm_stream stream);

/* incS ("incorrect segmentation"; DESIGN R26) of labels
 * against a phantom's truth: cluster j is mapped to the class of its centre's
 * rank (ascending, ties to the lower index; classes numbered by ascending
 * intensity level) and *count (dev int64) = the voxels whose mapped label
 * differs from the truth (exact integer).  labels, truth dev u8 [n];
 * centers dev fp32 [4].  Async. */
int pifcm_incs(pifcm_ctx *ctx, const uint8_t *labels, const uint8_t *truth, int64_t n, int32_t C,
               const float *centers, int64_t *count, pifcm_stream stream);
/* Eq. 11, host arithmetic: J[a] = 1/k sum_i alpha q_ia +
 * (1 - alpha) s_ia with q, s the incS and seconds of algorithm a at size i,
 * min-max normalised over the A algorithms at each size (a constant row
 * contributes 0).  incs, secs host [k][A]; J host [A].  PIFCM_EINVAL on bad
 * sizes or alpha outside [0, 1]. */
int pifcm_eq11(const double *incs, const double *secs, int32_t k, int32_t A, double alpha, double *J);

/* Defuzzification (R13): labels = argmax_j u_ij, ties to the
 * lowest j.  U dev fp32 [nz][ny][nx][4], labels dev u8.  Async. */
int pifcm_argmax(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t C, const float *U,
                 uint8_t *labels, pifcm_stream stream);

/* --------------------------------------------------------------- pipeline */
/* The whole method (Alg. 1 / Alg. 2): normalise,
 * histogram + GMM, FCM start (lambda = xi = 0) until eps, PSO over
 * (lambda, xi) with CHAINED fitness, final IFCM at the gbest from the gbest's
 * (U, c) until eps, argmax.  Sync.
 *   vol      dev [nz][ny][nx] of type dtype (PIFCM_U8, PIFCM_U16, PIFCM_F32)
 *   labels   dev u8 [nz][ny][nx]  out
 *   U_out    dev fp32 [nz][ny][nx][4] out, nullable: final memberships
 *   z_slice  -1: whole volume.  >= 0: the paper's `z` argument;
 *            the whole volume is segmented in 3D (R10) and only plane z_slice
 *            of `labels` is written (labels then points to [ny][nx]).
 *   rep      host out, nullable.
 * With a communicator attached (pifcm_ctx_dist, world > 1) the PSO is
 * particle-sharded: pso->p_begin / p_end must be this rank's
 * pifcm_dist_range (and ws sized for it); every rank returns the same labels
 * and report, bit-identical to the single-process call (CHAINED fitness).
 * Errors: as above, plus PIFCM_ENUMERIC for a non-finite fitness and
 * PIFCM_ENCCL for a failed collective. */
int pifcm_segment(pifcm_ctx *ctx, const void *vol, int32_t dtype, int32_t nx, int32_t ny,
                  int32_t nz, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                  int32_t z_slice, void *ws, size_t ws_bytes, uint8_t *labels, float *U_out,
                  pifcm_report *rep, pifcm_stream stream);

/* The literal slice mode (DESIGN R25; Alg. 1 with its input z, PAPER:93, 110:
 * "The z slice is assigned to a new variable"; the step runs
 * "through each voxel in the slice of a particular z axis image"): segment
 * slice z of a u8 volume with its 3D neighbourhood.  The volume is normalised
 * (Alg. 2 step 1); the R15 histogram of slice z on the volume's levels feeds
 * the GMM; FCM runs on the slice; the rows of planes z - v .. z - 1 and
 * z + 1 .. z + v (where they exist; v = the cfg's neighbourhood radius) are
 * the Eq. 2 memberships at the FCM centres and stay fixed; the CHAINED PSO
 * and the final IFCM update slice z only (Eq. 3 / Eq. 1 over the slice).
 * v = 1 .. 3, CHAINED, single process (eval_batch allowed).  Sync.
 *   vol     dev u8 [nz][ny][nx];  0 <= z < nz
 *   labels  dev u8 [ny][nx] out;  U_out dev fp32 [ny][nx][4] out, nullable
 *   ws      >= pifcm_segment_slice_workspace_size bytes (dev, 256-B aligned) */
int pifcm_segment_slice_workspace_size(int32_t nx, int32_t ny, int32_t nz, int32_t z, const pifcm_ifcm_cfg *cfg,
                                       const pifcm_pso_cfg *pso, size_t *bytes);
int pifcm_segment_slice(pifcm_ctx *ctx, const uint8_t *vol, int32_t nx, int32_t ny, int32_t nz, int32_t z,
                        const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes,
                        uint8_t *labels, float *U_out, pifcm_report *rep, pifcm_stream stream);

/* The same pipeline with HOST buffers (vol host u8, labels host u8): copies
 * the volume in, runs pifcm_segment, copies the labels out.  Sync. */
int pifcm_segment_host(pifcm_ctx *ctx, const uint8_t *vol_host, int32_t nx, int32_t ny,
                       int32_t nz, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                       void *ws, size_t ws_bytes, uint8_t *labels_host, pifcm_report *rep,
                       pifcm_stream stream);

/* ------------------------------------------------------------------- z-slab */
/* The IFCM step of a volume too large for one GPU, partitioned into z-slabs
 * across processes: per iteration the caller exchanges v halo
 * planes per neighbour and per state (pifcm_slab_halo_v + its own collective),
 * runs pifcm_slab_step, all-gathers the per-chunk partial records of all
 * ranks in rank order and calls pifcm_slab_finalize, which applies Eq. 3 /
 * Eq. 1 identically on every rank.  Because the records are
 * keyed by global z-chunks whose size depends on the volume alone
 * (pifcm_slab_chunk), centres and J are bit-identical for any number of
 * slabs, and equal to the single-GPU final IFCM of pifcm_segment, which runs
 * in the same decomposition. */

/* Planes per global z-chunk for a volume nx x ny x nz_total (host-only, no
 * GPU needed): every slab but the last holds a multiple of *tz planes and
 * starts at a multiple of *tz.  PIFCM_EINVAL on NULL / non-positive dims. */
int pifcm_slab_chunk(int32_t nx, int32_t ny, int32_t nz_total, int32_t *tz);

/* Partial records per state that pifcm_slab_step writes for this slab. */
int pifcm_slab_records(const pifcm_grid *grid, int32_t *nrec);

/* One Jacobi IFCM step over the slab's local planes for P
 * states, any v of cfg (v >= 2: the shell step, Eq. 9-10).  x dev fp32
 * [nz+2v][ny][pitch]; U_in, U_out dev fp32 [P][nz+2v][ny][nx][4] (halo planes
 * of U_in filled); centers dev fp32 [P][4]
 * (read only); lam_xi dev fp64 [P][2]; stats dev fp64 [P][4] nullable (states
 * with stats[p][3] != 0 are skipped); records dev fp64 [P][nrec][10] out:
 * per chunk and tile {sum u^m x (4), sum u^m (4), J, max|du|}.  Async. */
int pifcm_slab_step(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                    const float *x, const float *U_in, float *U_out, const float *centers,
                    const double *lam_xi, int32_t P, const double *stats, double *records,
                    pifcm_stream stream);

/* Eq. 3 / Eq. 1 from the gathered records [world][P][nrec][10] (rank order,
 * rank w's counts[w] <= nrec real records first, padding after; counts dev
 * int32 [world], nullable = all nrec; world <= 64): summed in canonical
 * (global chunk) order, then centres (kept where sum u^m < 1e-12, R9), stats
 * {J, max|du|, iterations += 1, converged = max|du| < eps} and fitness
 * (nullable).  Async. */
int pifcm_slab_finalize(pifcm_ctx *ctx, int32_t C, int32_t P, int32_t world, int32_t nrec,
                        const int32_t *counts, const double *records, float *centers, double *stats,
                        double *fitness, float eps, pifcm_stream stream);

/* The v halo planes per side of P slab states U [P][nz+2v][ny][nx][4]
 * (v = the cfg's neighbourhood radius, 1 .. 3):
 *   op 0: pack the first v local planes (array planes v .. 2v-1) into
 *         buf [P][v][ny][nx][4]
 *   op 1: pack the last v local planes (array planes nz .. nz+v-1) into buf
 *   op 2: unpack buf into the lower halo (array planes 0 .. v-1); zeros when
 *         z0 == 0
 *   op 3: unpack buf into the upper halo (planes nz+v .. nz+2v-1); zeros at
 *         the volume end
 * (buf may be NULL for a zero fill).  A slab thinner than v planes is only
 * valid at a volume end (PIFCM_EINVAL otherwise).  Async.
 * pifcm_slab_halo = pifcm_slab_halo_v with v = 1. */
int pifcm_slab_halo_v(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t v, int32_t P, int32_t op, float *U,
                      float *buf, pifcm_stream stream);
int pifcm_slab_halo(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t P, int32_t op, float *U,
                    float *buf, pifcm_stream stream);

/* ---------------------------------------- z-slab exchange over peer memory
 * The exchange steps of the slab iteration (halo planes, record gather)
 * done by the GPUs themselves over NVLink / NVSwitch peer mappings instead of
 * host-driven collectives: every rank allocates its two state buffers, two
 * gathered-record buffers and a flag word array with pifcm_peer_alloc,
 * exports them (pifcm_peer_handle, 64-byte CUDA IPC handles), opens the
 * other ranks' (pifcm_peer_open) and describes all of them in a
 * pifcm_peers.  pifcm_slab_p2p_run then runs the iterations with one device
 * barrier each and no host involvement between convergence checks. */
#define PIFCM_MAX_PEERS 16
typedef struct {
    int32_t world, rank;
    float *U[2][PIFCM_MAX_PEERS];      /* rank w's two state buffers [P][nz_w+2][ny][nx][4], this process's mapping */
    double *rec[2][PIFCM_MAX_PEERS];   /* rank w's gathered-record buffers [world][P][nrec_max][10] (even / odd epochs) */
    uint32_t *flags[PIFCM_MAX_PEERS];  /* rank w's words: [world] arrival epochs, [world] block counter, [world+1] status */
    int32_t nz[PIFCM_MAX_PEERS];       /* planes held by rank w */
} pifcm_peers;

/* Device memory that can be shared with other processes (cudaMalloc'ed,
 * zero-filled); free with pifcm_peer_free.  Sync. */
int pifcm_peer_alloc(pifcm_ctx *ctx, size_t bytes, void **ptr);
int pifcm_peer_free(pifcm_ctx *ctx, void *ptr);
/* 64-byte handle of an allocation of pifcm_peer_alloc (host out). */
int pifcm_peer_handle(pifcm_ctx *ctx, void *ptr, uint8_t *handle);
/* Map another process's allocation into this one; close with pifcm_peer_close. */
int pifcm_peer_open(pifcm_ctx *ctx, const uint8_t *handle, void **ptr);
int pifcm_peer_close(pifcm_ctx *ctx, void *ptr);

/* `iters` Jacobi IFCM iterations of P states over z-slab
 * ranks exchanging over peer memory.  Every rank calls it with the same
 * arguments except its slab.  The states start in the local planes of
 * U[*cur][rank] (their halo planes are filled here); after each step the
 * slab's boundary planes go straight into the neighbours' halo planes and
 * its records [P][nrec][10] (rec_local, scratch) into slot `rank` of every
 * rank's rec[epoch & 1]; after the device barrier (arrival epochs in the
 * flag words) each rank finalises Eq. 3 / Eq. 1 from its gathered buffer in
 * canonical order (as pifcm_slab_finalize with `counts`, dev int32 [world]).
 * The host checks convergence (stats, dev fp64 [P][4]) every 16 iterations.
 * On return *cur names the buffer holding the last iteration, *epoch the
 * next barrier epoch (pass it back on the next call), *iters_done the
 * iterations run.  A barrier that does not complete within ~20 s sets the
 * status word and the call returns PIFCM_ECUDA.  Sync. */
int pifcm_slab_p2p_run(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const float *x,
                       const pifcm_peers *peers, int32_t P, const int32_t *counts, int32_t nrec_max,
                       float *centers, const double *lam_xi, double *stats, double *rec_local, int32_t iters,
                       uint32_t *epoch, int32_t *cur, int32_t *iters_done, pifcm_stream stream);

/* ------------------------------------------- pipeline parts for z-slab ranks
 * Alg. 2 step 1 when the volume is split into slabs: each
 * rank reduces min / max over its own planes (pifcm_minmax_u8), the caller
 * combines them across ranks (min of mins, max of maxes), normalises its
 * slab arrays with the global range (pifcm_normalize_u8_range) and builds the
 * R15 histogram of its own planes (pifcm_hist_u8), which the caller sums
 * across ranks before pifcm_gmm_init.  All async. */
/* mm dev uint32 [2] out: {min, max} of the n u8 values at vol (dev). */
int pifcm_minmax_u8(pifcm_ctx *ctx, const uint8_t *vol, int64_t n, uint32_t *mm, pifcm_stream stream);
/* x = (v - mm[0]) / (mm[1] - mm[0]) (0 when mm[1] == mm[0], R16) for the
 * plain grid (nz_total = 0) vol [nz][ny][nx] -> x [nz][ny][pitch]. */
int pifcm_normalize_u8_range(pifcm_ctx *ctx, const pifcm_grid *grid, const uint8_t *vol, const uint32_t *mm,
                             float *x, pifcm_stream stream);
/* hist dev int64 [256] out: R15 bins b = round((v - min) * 255 / (max - min))
 * of the n values at vol, with the global range mm. */
int pifcm_hist_u8(pifcm_ctx *ctx, const uint8_t *vol, int64_t n, const uint32_t *mm, int64_t *hist,
                  pifcm_stream stream);

/* ------------------------------------------------- PSO over z-slab ranks
 * Alg. 1 steps 3-10 for a volume split into z-slabs (SURVEY
 * 8(e), the 512^3 C5 workload): every rank holds ALL particles' states for
 * its slab (a slot pool like pifcm_pso_*, each slot [nz+2v][ny][nx][4] with
 * the halo planes) and the identical swarm.  Per generation the caller runs
 *   pifcm_slab_pso_halo (pack, op 0/1) -> send/recv -> pifcm_slab_pso_halo
 *   (unpack, op 2/3) -> pifcm_slab_pso_eval (records of every particle) ->
 *   all-gather of the records in rank order -> pifcm_slab_pso_finalize
 *   (centres and fitness of every particle, identical on every rank) ->
 *   pifcm_slab_pso_update (the device PSO update of pifcm_pso_update)
 * so every rank takes the same PSO decisions; fitness and trajectories are
 * bit-identical for any number of slabs (global z-chunk records).  `slab` is
 * the rank's slab grid (see pifcm_grid); pso->p_begin = p_end = 0 (all
 * particles).  The workspace holds the slots, the swarm and scratch. */
int pifcm_slab_workspace_size(const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                              size_t *bytes);
/* U0 dev fp32 [nz+2v][ny][nx][4] (the slab's start state, halos included),
 * c0 dev fp32 [4].  Positions / velocities from Philox (R12).  Async. */
int pifcm_slab_pso_init(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                        const float *U0, const float *c0, void *ws, size_t ws_bytes, pifcm_stream stream);
/* Halo planes of every particle's current state, ops as pifcm_slab_halo_v
 * with the cfg's v and buf [P][v][ny][nx][4].  Async. */
int pifcm_slab_pso_halo(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                        void *ws, size_t ws_bytes, int32_t op, float *buf, pifcm_stream stream);
/* One IFCM step of every particle at its own (lambda, xi) on the slab's
 * planes (Alg. 1 step 4, CHAINED R11); records dev fp64 [P][nrec][10] out
 * (nrec = pifcm_slab_records).  x dev fp32 [nz+2v][ny][pitch].  Async. */
int pifcm_slab_pso_eval(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                        const float *x, void *ws, size_t ws_bytes, double *records, pifcm_stream stream);
/* Eq. 3 / Eq. 1 of every particle from the gathered records [world][P][nrec][10]
 * (as pifcm_slab_finalize) into the swarm's centres and fitness.  Async. */
int pifcm_slab_pso_finalize(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                            const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes, int32_t world, int32_t nrec,
                            const int32_t *counts, const double *records, pifcm_stream stream);
/* Alg. 1 steps 5-8 (as pifcm_pso_update).  Async. */
int pifcm_slab_pso_update(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                          const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes, pifcm_stream stream);
/* As pifcm_pso_result_get / pifcm_pso_gbest_state (U_out: the slab part of
 * the gbest state, [nz+2v][ny][nx][4]; every rank holds it).  Sync. */
int pifcm_slab_pso_result_get(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                              const pifcm_pso_cfg *pso, void *ws, pifcm_pso_result *out, int32_t *stopped,
                              pifcm_stream stream);
int pifcm_slab_pso_gbest_state(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                               const pifcm_pso_cfg *pso, void *ws, float *U_out, float *c_out, pifcm_stream stream);

/* Number of kernels this context has launched so far (for the bench's
 * gpu_launches count). */
int64_t pifcm_launch_count(const pifcm_ctx *ctx);

/* Device timing of the fused step kernel: when enabled (which resets the
 * counters), every launch of the neighbourhood (stencil) step kernel is
 * bracketed by CUDA events on its stream.  pifcm_timing_read synchronises
 * those events and returns, for the batched launches (batched = 1: P > 1
 * states per launch, i.e. the PSO generations) or the single-state launches
 * (batched = 0: the final IFCM), the summed kernel time in ms, the number of
 * launches and their algorithmic bytes (per launch: P * nvox * 32 bytes of
 * AoS-C4 membership read + write, plus nvox * 4 bytes of intensities). */
int pifcm_timing_enable(pifcm_ctx *ctx, int32_t on);
int pifcm_timing_read(pifcm_ctx *ctx, int32_t batched, double *ms_total, int64_t *launches,
                      double *alg_bytes);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* PIFCM_H */
