// host.cu -- the C ABI of libpifcm.so (include/pifcm.h): validation, workspace
// layout and orchestration of the kernels in step.cu / aux_kernels.cu.
// Everything on the path runs in those kernels; this file only launches.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <cmath>

#include <chrono>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "pifcm_comm.h"
#include "pifcm_internal.cuh"

using namespace pifcm;

struct pifcm_ctx {
    int device = 0;
    std::string err = "ok";
    long long launches = 0;
    cudaEvent_t ev[8];
    // fused-step timing (pifcm_timing_*)
    bool timing = false;
    std::vector<cudaEvent_t> tev;   // pairs (start, stop)
    std::vector<int> tcls;          // class of each pair: 0 batched (P > 1), 1 single state
    size_t tused = 0;               // events in use
    double t_ms[2] = {0.0, 0.0}, t_bytes[2] = {0.0, 0.0};
    long long t_launches[2] = {0, 0};
    pifcm::Comm comm;  // pifcm_ctx_dist
    // pifcm_pso_trace
    double *tr_f = nullptr, *tr_pos = nullptr;
    int *tr_gbest = nullptr;
    int tr_max = 0;
};

namespace {

int fail(pifcm_ctx *ctx, int code, const char *fmt, ...) {
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        ctx->err = buf;
    }
    return code;
}

#define CK(ctx, expr)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail((ctx), PIFCM_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                              \
    } while (0)

// Every launch goes to the context's device (a process may hold contexts on
// several devices; cudaSetDevice is a no-op when it is already current).
#define LAUNCH(ctx, n, expr)                        \
    do {                                            \
        CK(ctx, cudaSetDevice((ctx)->device));      \
        CK(ctx, expr);                              \
        (ctx)->launches += (n);                     \
    } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int check_grid(pifcm_ctx *ctx, const pifcm_grid *g) {
    if (!g) return fail(ctx, PIFCM_EINVAL, "grid is NULL");
    if (g->nx < 1 || g->ny < 1 || g->nz < 1)
        return fail(ctx, PIFCM_EINVAL, "grid dims must be >= 1 (got %d x %d x %d)", g->nx, g->ny, g->nz);
    if (g->pitch < g->nx) return fail(ctx, PIFCM_EINVAL, "pitch %d < nx %d", g->pitch, g->nx);
    if (g->pitch % 4 != 0) return fail(ctx, PIFCM_EALIGN, "pitch %d is not a multiple of 4", g->pitch);
    const bool slab = g->nz_total > 0 && !(g->z0 == 0 && g->nz_total == g->nz);
    if (slab) return fail(ctx, PIFCM_EINVAL, "z-slab grids (nz_total > 0) are only for the pifcm_slab_* calls");
    if ((long long)g->nx * g->ny * g->nz >= (1LL << 31))
        return fail(ctx, PIFCM_EINVAL, "volume of %lld voxels >= 2^31 (use z-slab sharding)",
                    (long long)g->nx * g->ny * g->nz);
    return PIFCM_OK;
}

int check_cfg(pifcm_ctx *ctx, const pifcm_ifcm_cfg *c) {
    if (!c) return fail(ctx, PIFCM_EINVAL, "cfg is NULL");
    if (c->C < 2 || c->C > kMaxC) return fail(ctx, PIFCM_EINVAL, "C = %d outside [2, 4]", c->C);
    if (!(c->m > 1.0f) || !(c->m < 1e6f)) return fail(ctx, PIFCM_EINVAL, "m = %g must be > 1", (double)c->m);
    if (c->v < 1 || c->v > kMaxV) return fail(ctx, PIFCM_EINVAL, "v = %d: the device path has v = 1 .. %d", c->v, kMaxV);
    if (!(c->h > 0.0f)) return fail(ctx, PIFCM_EINVAL, "h must be > 0");
    if (c->q_mode != PIFCM_Q_LITERAL && c->q_mode != PIFCM_Q_SQEUCLID)
        return fail(ctx, PIFCM_EINVAL, "q_mode %d unknown", c->q_mode);
    if (c->max_iter < 1) return fail(ctx, PIFCM_EINVAL, "max_iter must be >= 1");
    return PIFCM_OK;
}

int check_pso(pifcm_ctx *ctx, const pifcm_pso_cfg *p) {
    if (!p) return fail(ctx, PIFCM_EINVAL, "pso cfg is NULL");
    if (p->P < 1 || p->P > 1024) return fail(ctx, PIFCM_EINVAL, "P = %d outside [1, 1024]", p->P);
    if (p->ring_k < 0) return fail(ctx, PIFCM_EINVAL, "ring_k must be >= 0");
    if (p->max_gen < 1) return fail(ctx, PIFCM_EINVAL, "max_gen must be >= 1");
    if (!(p->vmax > 0.0) || !(p->v0 >= 0.0)) return fail(ctx, PIFCM_EINVAL, "vmax > 0, v0 >= 0 required");
    if (p->fitness_mode < PIFCM_FIT_CHAINED || p->fitness_mode > PIFCM_FIT_LEADER)
        return fail(ctx, PIFCM_EINVAL, "fitness_mode %d unknown", p->fitness_mode);
    if (p->fitness_mode != PIFCM_FIT_CHAINED && p->P > 128)
        return fail(ctx, PIFCM_EINVAL, "ANCHORED / LEADER fitness supports P <= 128");
    const bool all = (p->p_begin == 0 && p->p_end == 0);
    if (!all && (p->p_begin < 0 || p->p_end > p->P || p->p_begin >= p->p_end))
        return fail(ctx, PIFCM_EINVAL, "particle range [%d, %d) invalid for P = %d", p->p_begin, p->p_end, p->P);
    return PIFCM_OK;
}

// mode / shell combinations the device path implements
int check_pso_cfg(pifcm_ctx *ctx, const pifcm_ifcm_cfg *c, const pifcm_pso_cfg *p) {
    (void)ctx; (void)c; (void)p;  // every fitness mode runs with v = 1 and v = 2
    return PIFCM_OK;
}

void prange(const pifcm_pso_cfg *p, int *p0, int *pl) {
    if (p->p_begin == 0 && p->p_end == 0) { *p0 = 0; *pl = p->P; }
    else { *p0 = p->p_begin; *pl = p->p_end - p->p_begin; }
}

// Scratch of the value-histogram FCM: x, count and previous row per value.
size_t fcm_hist_ws_bytes(int nvals) {
    return align_up(sizeof(float) * nvals, 256) + align_up(sizeof(double) * nvals, 256) +
           align_up(sizeof(float4) * nvals, 256);
}
FcmHistArgs fcm_hist_args(void *ws, int nvals) {
    FcmHistArgs a{};
    char *b = static_cast<char *>(ws);
    a.nvals = nvals;
    a.xs = reinterpret_cast<float *>(b);
    b += align_up(sizeof(float) * nvals, 256);
    a.ns = reinterpret_cast<double *>(b);
    b += align_up(sizeof(double) * nvals, 256);
    a.up = reinterpret_cast<float4 *>(b);
    return a;
}

// Workspace layout (all offsets 256-byte aligned).
struct Layout {
    size_t x, vol, lab, hist, mm, c0, slots, hdr, dhdr, pos, vel, pbf, pbx, fit, evalpos, cur, nxt,
        gbc, cent, part, stats, lamxi, cnt, gbar, hf, shc, vcnt, fhws, cprev, fstats, total;
    int nslots, P, Pl, p0, nblk, mode, eb;  // eb: states per evaluation launch (CHAINED)
    long long nvox;
};

Layout layout(const pifcm_grid *g, const pifcm_ifcm_cfg *c, const pifcm_pso_cfg *pso) {
    (void)c;
    Layout L{};
    L.nvox = (long long)g->nx * g->ny * g->nz;
    int P = 1, p0 = 0, Pl = 1;
    if (pso) { P = pso->P; prange(pso, &p0, &Pl); }
    L.P = P; L.Pl = Pl; L.p0 = p0;
    L.mode = pso ? pso->fitness_mode : PIFCM_FIT_CHAINED;
    // CHAINED: every particle's state, the slot its next evaluation writes and
    // the pinned gbest; ANCHORED: the shared start + the gbest snapshot;
    // LEADER: the shared state, its successor and the pinned gbest
    // (batched CHAINED evaluation: every particle's state, one batch of new
    // states, the pinned gbest)
    L.eb = (pso && pso->eval_batch > 0 && pso->eval_batch < Pl) ? pso->eval_batch : Pl;
    L.nslots = L.mode == PIFCM_FIT_CHAINED ? (L.eb < Pl ? Pl + L.eb + 1 : 2 * Pl + 1)
                                           : (L.mode == PIFCM_FIT_LEADER ? 3 : 2);
    L.nblk = step_nblk_max(g->nx, g->ny, g->nz);
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
    L.x = take(sizeof(float) * (size_t)g->pitch * g->ny * g->nz);
    L.vol = take((size_t)L.nvox);
    L.lab = take((size_t)L.nvox);
    L.hist = take(sizeof(int64_t) * 256);
    L.mm = take(sizeof(unsigned int) * 2);
    L.c0 = take(sizeof(float) * 4);
    L.slots = take(sizeof(float4) * (size_t)L.nvox * L.nslots);
    L.hdr = take(sizeof(int) * 16);
    L.dhdr = take(sizeof(double) * 16);
    L.pos = take(sizeof(double) * 2 * P);
    L.vel = take(sizeof(double) * 2 * P);
    L.pbf = take(sizeof(double) * P);
    L.pbx = take(sizeof(double) * 2 * P);
    L.fit = take(sizeof(double) * P);
    L.evalpos = take(sizeof(double) * 2 * P);
    L.cur = take(sizeof(int) * Pl);
    L.nxt = take(sizeof(int) * Pl);
    L.gbc = take(sizeof(float) * 4);
    L.cent = take(sizeof(float) * 4 * (Pl > 2 ? Pl : 2));
    {
        size_t np = (size_t)kNR * L.nblk * (Pl > 1 ? Pl : 1);
        const size_t ne = (size_t)eval_shared_parts(L.nvox, Pl) * Pl;
        L.part = take(sizeof(double) * (np > ne ? np : ne));
    }
    L.stats = take(sizeof(double) * 4 * (Pl > 1 ? Pl : 1));
    L.lamxi = take(sizeof(double) * 2 * (Pl > 1 ? Pl : 1));
    L.cnt = take(sizeof(unsigned) * (Pl > 1 ? Pl : 1));
    L.gbar = take(sizeof(unsigned) * 3);  // grid barrier + release word of the 2D final-IFCM loop
    L.hf = L.mode == PIFCM_FIT_CHAINED ? take(0) : take(sizeof(float4) * 2 * (size_t)L.nvox);
    L.shc = take(sizeof(float) * 4);
    // the FCM start on the value histogram (any quantised dtype)
    L.vcnt = take(sizeof(int64_t) * 65536);
    L.fhws = take(fcm_hist_ws_bytes(65536));
    L.cprev = take(sizeof(float) * 4);
    L.fstats = take(sizeof(double) * 4);
    L.total = o;
    return L;
}

template <typename T>
T *at(void *ws, size_t off) { return reinterpret_cast<T *>(static_cast<char *>(ws) + off); }

SwarmDev swarm_of(void *ws, const Layout &L) {
    SwarmDev s;
    s.hdr = at<int>(ws, L.hdr);
    s.dhdr = at<double>(ws, L.dhdr);
    s.pos = at<double>(ws, L.pos);
    s.vel = at<double>(ws, L.vel);
    s.pbf = at<double>(ws, L.pbf);
    s.pbx = at<double>(ws, L.pbx);
    s.fit = at<double>(ws, L.fit);
    s.evalpos = at<double>(ws, L.evalpos);
    s.cur = at<int>(ws, L.cur);
    s.nxt = at<int>(ws, L.nxt);
    s.gbest_c = at<float>(ws, L.gbc);
    s.centers = at<float>(ws, L.cent);
    return s;
}

int check_ws(pifcm_ctx *ctx, void *ws, size_t ws_bytes, size_t need) {
    if (need > 0 && !ws) return fail(ctx, PIFCM_EINVAL, "workspace is NULL");
    if (ws_bytes < need) return fail(ctx, PIFCM_ENOMEM, "workspace %zu bytes < required %zu", ws_bytes, need);
    if (ws && (reinterpret_cast<uintptr_t>(ws) & 255u))
        return fail(ctx, PIFCM_EALIGN, "workspace must be 256-byte aligned");
    return PIFCM_OK;
}

// Eq. 10 shell weights W_r = e^{-r/h} / sum_{s=1..v} e^{-s/h}.
void set_shells(StepArgs &a, const pifcm_ifcm_cfg *cfg) {
    a.v = cfg->v;
    double s = 0.0;
    for (int r = 1; r <= cfg->v; ++r) s += exp(-(double)r / (double)cfg->h);
    for (int r = 1; r <= kMaxV; ++r) {  // Eq. 10
        a.wshd[r - 1] = r <= cfg->v ? exp(-(double)r / (double)cfg->h) / s : 0.0;
        a.wsh[r - 1] = (float)a.wshd[r - 1];
    }
}

// A step launch, bracketed by CUDA events on its stream when timing is on
// (stencil launches only; vox = the voxels the launch updates per state).
int timed_step(pifcm_ctx *ctx, const StepArgs &a, int C, bool stencil, int P, long long vox, cudaStream_t st) {
    const bool timed = ctx->timing && stencil;
    if (timed) {
        while (ctx->tev.size() < ctx->tused + 2) {
            cudaEvent_t e;
            CK(ctx, cudaEventCreate(&e));
            ctx->tev.push_back(e);
        }
        CK(ctx, cudaEventRecord(ctx->tev[ctx->tused], st));
    }
    LAUNCH(ctx, 1, launch_step(a, C, stencil, P, st));
    if (timed) {
        CK(ctx, cudaEventRecord(ctx->tev[ctx->tused + 1], st));
        const int cls = P > 1 ? 0 : 1;
        if (ctx->tcls.size() < ctx->tused / 2 + 1) ctx->tcls.resize(ctx->tused / 2 + 1);
        ctx->tcls[ctx->tused / 2] = cls;
        ctx->tused += 2;
        ctx->t_bytes[cls] += 32.0 * (double)vox * P + 4.0 * (double)vox;
        ctx->t_launches[cls] += 1;
    }
    return PIFCM_OK;
}

// The arguments of a step launch for P states.
StepArgs step_args(const pifcm_grid *g, const pifcm_ifcm_cfg *cfg, const float *x, const float4 *Uin,
                   float4 *Uout, const int *in_idx, const int *out_idx, float *centers, const double *lamxi,
                   int first, double *partials, double *fitness, double *stats, float eps, int *status,
                   const int *stop, int n_in_states, unsigned *counters, bool canonical) {
    StepArgs a{};
    a.x = x;
    a.nx = g->nx; a.ny = g->ny; a.nz = g->nz; a.pitch = g->pitch;
    a.nvox = (long long)g->nx * g->ny * g->nz;
    a.U_in = Uin; a.U_out = Uout; a.in_idx = in_idx; a.out_idx = out_idx;
    a.centers = centers; a.lam_xi = lamxi; a.partials = partials;
    a.stats = stats; a.stop = stop;
    a.m = cfg->m; a.inv_m1 = 1.0f / (cfg->m - 1.0f);
    a.q_mode = cfg->q_mode; a.first = first;
    set_shells(a, cfg);
    a.n_in_states = n_in_states;
    a.want_du = (stats != nullptr) ? 1 : 0;
    a.counters = counters;
    a.canonical = canonical ? 1 : 0;
    a.C = cfg->C;
    a.fitness = fitness;
    a.stats_out = stats;
    a.eps = eps;
    a.status = status;
    return a;
}

// One step launch + finalize for P states.
int run_step(pifcm_ctx *ctx, const pifcm_grid *g, const pifcm_ifcm_cfg *cfg, const float *x,
             const float4 *Uin, float4 *Uout, const int *in_idx, const int *out_idx,
             float *centers, const double *lamxi, bool stencil, int first, int P,
             double *partials, double *fitness, double *stats, float eps, int *status,
             const int *stop, cudaStream_t st, int n_in_states, unsigned *counters, bool canonical = false) {
    const StepArgs a = step_args(g, cfg, x, Uin, Uout, in_idx, out_idx, centers, lamxi, first, partials, fitness,
                                 stats, eps, status, stop, n_in_states, counters, canonical);
    int r = timed_step(ctx, a, cfg->C, stencil, P, a.nvox, st);
    if (r) return r;
    // Eq. 3 / Eq. 1 finalisation is fused: the last CTA of each state sums the
    // partial records (finalize_if_last in step.cu) -- in the canonical
    // decomposition exactly as k_slab_finalize sums the records of a slab split
    return PIFCM_OK;
}

// The iterations of one 2D state (nz = 1, v = 1) in one cooperative launch
// (k_step_2d_loop: a grid barrier and the canonical finalisation between the
// steps, the same records and sums as one launch per step, so the results are
// bit-identical).  *used = false when it did not run (not 2D, or its CTAs
// cannot all be resident): the caller then launches per step.  The iterations
// run are stats[2] (read by the caller, who also passes them to
// loop_timing_count when timing is on).
int run_2d_loop(pifcm_ctx *ctx, const pifcm_grid *g, const pifcm_ifcm_cfg *cfg, const float *x, float4 *UA,
                float4 *UB, float *centers, const double *lamxi, int iters, double *partials, double *stats,
                int *status, unsigned *counters, unsigned *gbar, cudaStream_t st, bool *used) {
    *used = false;
    if (g->nz != 1 || g->nz_total > 1 || cfg->v != 1 || iters < 2 || !gbar || !stats) return PIFCM_OK;
    const StepArgs a = step_args(g, cfg, x, UA, UB, nullptr, nullptr, centers, lamxi, 0, partials, nullptr, stats,
                                 cfg->eps, status, nullptr, 1, counters, true);
    const bool timed = ctx->timing;
    if (timed) {
        while (ctx->tev.size() < ctx->tused + 2) {
            cudaEvent_t e;
            CK(ctx, cudaEventCreate(&e));
            ctx->tev.push_back(e);
        }
        CK(ctx, cudaEventRecord(ctx->tev[ctx->tused], st));
    }
    LAUNCH(ctx, 1, launch_2d_loop(a, cfg->C, UA, UB, iters, gbar, st, used));
    if (timed) {
        CK(ctx, cudaEventRecord(ctx->tev[ctx->tused + 1], st));
        if (ctx->tcls.size() < ctx->tused / 2 + 1) ctx->tcls.resize(ctx->tused / 2 + 1);
        ctx->tcls[ctx->tused / 2] = 1;  // single-state class; launches / bytes added by loop_timing_count
        ctx->tused += 2;
    }
    return PIFCM_OK;
}
// Count the iterations of a run_2d_loop launch as single-state launches.
void loop_timing_count(pifcm_ctx *ctx, int done, long long vox) {
    if (!ctx->timing) return;
    ctx->t_bytes[1] += 36.0 * (double)vox * done;
    ctx->t_launches[1] += done;
}

// lambda = xi = 0 exactly -> the pointwise FCM kernel (Eq. 4 reduces to the plain distance).
bool host_zero_lamxi(const double *lamxi_dev, int P, cudaStream_t st, bool *ok) {
    double buf[2 * 64];
    if (P > 64) { *ok = true; return false; }
    if (cudaMemcpyAsync(buf, lamxi_dev, sizeof(double) * 2 * P, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) { *ok = false; return false; }
    *ok = true;
    for (int i = 0; i < 2 * P; ++i)
        if (buf[i] != 0.0) return false;
    return true;
}

}  // namespace

// ============================================================== ABI: context
extern "C" {

const char *pifcm_version(void) { return "pifcm-b200 0.1 (sm_100a)"; }

int pifcm_ctx_create(int device, pifcm_ctx **out) {
    if (!out) return PIFCM_EINVAL;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return PIFCM_ECUDA;
    if (cudaSetDevice(device) != cudaSuccess) return PIFCM_ECUDA;
    pifcm_ctx *c = new pifcm_ctx();
    c->device = device;
    for (int i = 0; i < 8; ++i)
        if (cudaEventCreate(&c->ev[i]) != cudaSuccess) { delete c; return PIFCM_ECUDA; }
    *out = c;
    return PIFCM_OK;
}

void pifcm_ctx_destroy(pifcm_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    pifcm::comm_free(ctx->comm);
    for (int i = 0; i < 8; ++i) cudaEventDestroy(ctx->ev[i]);
    for (cudaEvent_t e : ctx->tev) cudaEventDestroy(e);
    delete ctx;
}

const char *pifcm_last_error(const pifcm_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int pifcm_nccl_unique_id(uint8_t id[128]) {
    if (!id) return PIFCM_EINVAL;
    std::string err;
    return pifcm::comm_unique_id(id, err);
}

int pifcm_ctx_dist(pifcm_ctx *ctx, const pifcm_dist *dist, const pifcm_host_coll *coll) {
    if (!ctx) return PIFCM_EINVAL;
    if (!dist) return fail(ctx, PIFCM_EINVAL, "dist is NULL");
    if (dist->world < 1) return fail(ctx, PIFCM_EINVAL, "world = %d < 1", dist->world);
    std::string err;
    const int r = pifcm::comm_init(ctx->comm, ctx->device, dist, coll, err);
    return r ? fail(ctx, r, "pifcm_ctx_dist: %s", err.c_str()) : PIFCM_OK;
}

int pifcm_dist_range(int32_t P, int32_t world, int32_t rank, int32_t *p_begin, int32_t *p_end) {
    if (!p_begin || !p_end || P < 1 || world < 1 || rank < 0 || rank >= world) return PIFCM_EINVAL;
    int a, b;
    pifcm::dist_range(P, world, rank, &a, &b);
    *p_begin = a;
    *p_end = b;
    return PIFCM_OK;
}

int64_t pifcm_launch_count(const pifcm_ctx *ctx) { return ctx ? ctx->launches : 0; }

static int timing_drain(pifcm_ctx *ctx) {
    for (size_t i = 0; i + 1 < ctx->tused; i += 2) {
        CK(ctx, cudaEventSynchronize(ctx->tev[i + 1]));
        float ms = 0.f;
        CK(ctx, cudaEventElapsedTime(&ms, ctx->tev[i], ctx->tev[i + 1]));
        ctx->t_ms[ctx->tcls[i / 2]] += ms;
    }
    ctx->tused = 0;
    return PIFCM_OK;
}

int pifcm_timing_enable(pifcm_ctx *ctx, int32_t on) {
    if (!ctx) return PIFCM_EINVAL;
    int r = timing_drain(ctx);
    if (r) return r;
    ctx->timing = on != 0;
    for (int c = 0; c < 2; ++c) {
        ctx->t_ms[c] = 0.0;
        ctx->t_bytes[c] = 0.0;
        ctx->t_launches[c] = 0;
    }
    return PIFCM_OK;
}

int pifcm_timing_read(pifcm_ctx *ctx, int32_t batched, double *ms_total, int64_t *launches, double *alg_bytes) {
    if (!ctx || batched < 0 || batched > 1) return PIFCM_EINVAL;
    int r = timing_drain(ctx);
    if (r) return r;
    const int c = batched ? 0 : 1;
    if (ms_total) *ms_total = ctx->t_ms[c];
    if (launches) *launches = ctx->t_launches[c];
    if (alg_bytes) *alg_bytes = ctx->t_bytes[c];
    return PIFCM_OK;
}

int pifcm_workspace_size(const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                         size_t *bytes) {
    if (!bytes) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(nullptr, grid)) || (r = check_cfg(nullptr, cfg))) return r;
    if (pso && ((r = check_pso(nullptr, pso)) || (r = check_pso_cfg(nullptr, cfg, pso)))) return r;
    *bytes = layout(grid, cfg, pso).total;
    return PIFCM_OK;
}

int pifcm_iterate_workspace_size(const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, int32_t P,
                                 int32_t iters, size_t *bytes) {
    if (!bytes) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(nullptr, grid)) || (r = check_cfg(nullptr, cfg))) return r;
    if (P < 1 || iters < 1) return PIFCM_EINVAL;
    const long long nvox = (long long)grid->nx * grid->ny * grid->nz;
    const int nblk = step_nblk_max(grid->nx, grid->ny, grid->nz);
    size_t b = align_up(sizeof(double) * kNR * (size_t)nblk * P, 256) +  // partials
               align_up(sizeof(double) * 4 * P, 256) + 256 +             // stats scratch + status
               align_up(sizeof(unsigned) * P, 256) + 256;                // finalisation counters, grid barrier
    if (iters > 1) b += align_up(sizeof(float4) * (size_t)nvox * P, 256);
    *bytes = b;
    return PIFCM_OK;
}

// ============================================================== ABI: iterate
int pifcm_iterate(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const float *x,
                  const float *U_in, float *U_out, float *centers, const double *lam_xi, int32_t P,
                  int32_t iters, double *stats, void *ws, size_t ws_bytes, pifcm_stream stream) {
    return pifcm_iterate_ex(ctx, grid, cfg, x, U_in, U_out, centers, lam_xi, P, iters, stats, ws, ws_bytes, 0,
                            stream);
}

int pifcm_iterate_ex(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const float *x,
                     const float *U_in, float *U_out, float *centers, const double *lam_xi, int32_t P,
                     int32_t iters, double *stats, void *ws, size_t ws_bytes, int32_t flags,
                     pifcm_stream stream) {
    if (flags & ~(PIFCM_ITER_CANONICAL | PIFCM_ITER_PER_STEP))
        return ctx ? fail(ctx, PIFCM_EINVAL, "unknown flags %d", flags) : PIFCM_EINVAL;
    const bool canonical = (flags & PIFCM_ITER_CANONICAL) != 0;
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid)) || (r = check_cfg(ctx, cfg))) return r;
    if (P < 1 || P > 65535) return fail(ctx, PIFCM_EINVAL, "P = %d outside [1, 65535]", P);
    if (iters < 1) return fail(ctx, PIFCM_EINVAL, "iters must be >= 1");
    if (!x || !U_in || !U_out || !centers || !lam_xi)
        return fail(ctx, PIFCM_EINVAL, "x, U_in, U_out, centers and lam_xi must be non-NULL");
    if (U_in == U_out) return fail(ctx, PIFCM_EINVAL, "U_in and U_out must not alias");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(U_in) |
         reinterpret_cast<uintptr_t>(U_out)) & 15u)
        return fail(ctx, PIFCM_EALIGN, "x, U_in and U_out must be 16-byte aligned");
    size_t need = 0;
    pifcm_iterate_workspace_size(grid, cfg, P, iters, &need);
    if ((r = check_ws(ctx, ws, ws_bytes, need))) return r;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CK(ctx, cudaSetDevice(ctx->device));
    const long long nvox = (long long)grid->nx * grid->ny * grid->nz;
    const int nblk = step_nblk_max(grid->nx, grid->ny, grid->nz);
    size_t o = 0;
    double *partials = at<double>(ws, o); o = align_up(o + sizeof(double) * kNR * (size_t)nblk * P, 256);
    double *st_scr = at<double>(ws, o); o = align_up(o + sizeof(double) * 4 * P, 256);
    int *status = at<int>(ws, o); o += 256;
    unsigned *counters = at<unsigned>(ws, o); o = align_up(o + sizeof(unsigned) * P, 256);
    unsigned *gbar = at<unsigned>(ws, o); o += 256;
    float4 *scratch = iters > 1 ? at<float4>(ws, o) : nullptr;
    CK(ctx, cudaMemsetAsync(counters, 0, sizeof(unsigned) * P, st));
    double *S = stats ? stats : st_scr;
    CK(ctx, cudaMemsetAsync(S, 0, sizeof(double) * 4 * P, st));
    CK(ctx, cudaMemsetAsync(status, 0, sizeof(int), st));
    // a small 2D image (C1): all iterations in one launch, one CTA per state
    // holding the image in shared memory (small2d.cu); not for the canonical
    // decomposition, whose records must match the pipeline's final IFCM
    if (!canonical && cfg->v == 1 && grid->nz == 1 && (long long)grid->nx * grid->ny <= 4096 &&
        small2d_smem(grid->nx, grid->ny) <= 200 * 1024) {
        LAUNCH(ctx, 1, launch_iterate_small2d(x, grid->nx, grid->ny, grid->pitch, reinterpret_cast<const float4 *>(U_in),
                                              reinterpret_cast<float4 *>(U_out), centers, lam_xi, P, iters,
                                              cfg->eps, cfg->m, cfg->q_mode, cfg->C, S, status, st));
        return PIFCM_OK;
    }
    bool ok = true;
    const bool zero = host_zero_lamxi(lam_xi, P, st, &ok);
    if (!ok) return fail(ctx, PIFCM_ECUDA, "reading lam_xi failed");
    const float eps = cfg->eps;
    if (canonical && !zero && P == 1 && iters > 1 && !(flags & PIFCM_ITER_PER_STEP)) {
        // a 2D image: every iteration in one cooperative launch (bit-identical
        // to one launch per step); buffers ordered so that, as below, step t
        // writes U_out iff iters - t is even (launch_fixup_copy's convention)
        float4 *Uo = reinterpret_cast<float4 *>(U_out);
        float4 *UA = (iters & 1) ? scratch : Uo, *UB = (iters & 1) ? Uo : scratch;
        bool used = false;
        if (grid->nz == 1 && cfg->v == 1) {
            CK(ctx, cudaMemcpyAsync(UA, U_in, sizeof(float4) * (size_t)nvox, cudaMemcpyDeviceToDevice, st));
            if ((r = run_2d_loop(ctx, grid, cfg, x, UA, UB, centers, lam_xi, iters, partials, S, status, counters,
                                 gbar, st, &used)))
                return r;
        }
        if (used) {
            loop_timing_count(ctx, iters, nvox);
            if (eps > 0.f) LAUNCH(ctx, 1, launch_fixup_copy(scratch, Uo, nvox, P, S, iters, st));
            return PIFCM_OK;
        }
    }
    const float4 *src = reinterpret_cast<const float4 *>(U_in);
    for (int t = 1; t <= iters; ++t) {
        float4 *dst = (((iters - t) & 1) == 0) ? reinterpret_cast<float4 *>(U_out) : scratch;
        r = run_step(ctx, grid, cfg, x, src, dst, nullptr, nullptr, centers, lam_xi, !zero, 0, P,
                     partials, nullptr, S, eps, status, nullptr, st, P, counters, canonical && !zero);
        if (r) return r;
        src = dst;
    }
    if (eps > 0.f && iters > 1)
        LAUNCH(ctx, 1, launch_fixup_copy(scratch, reinterpret_cast<float4 *>(U_out), nvox, P, S, iters, st));
    return PIFCM_OK;
}

// ============================================================== ABI: PSO
static int pso_common(pifcm_ctx *ctx, const pifcm_grid *g, const pifcm_ifcm_cfg *c, const pifcm_pso_cfg *p,
                      void *ws, size_t ws_bytes, Layout *L) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, g)) || (r = check_cfg(ctx, c)) || (r = check_pso(ctx, p)) ||
        (r = check_pso_cfg(ctx, c, p)))
        return r;
    *L = layout(g, c, p);
    CK(ctx, cudaSetDevice(ctx->device));
    return check_ws(ctx, ws, ws_bytes, L->total);
}

int pifcm_pso_init(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                   const float *U0, const float *c0, void *ws, size_t ws_bytes, pifcm_stream stream) {
    Layout L;
    int r = pso_common(ctx, grid, cfg, pso, ws, ws_bytes, &L);
    if (r) return r;
    if (!U0 || !c0) return fail(ctx, PIFCM_EINVAL, "U0 and c0 must be non-NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CK(ctx, cudaSetDevice(ctx->device));
    float4 *slot0 = at<float4>(ws, L.slots);
    if (reinterpret_cast<const void *>(U0) != slot0)
        CK(ctx, cudaMemcpyAsync(slot0, U0, sizeof(float4) * (size_t)L.nvox, cudaMemcpyDeviceToDevice, st));
    const uint32_t k0 = (uint32_t)(pso->seed & 0xFFFFFFFFu), k1 = (uint32_t)(pso->seed >> 32);
    CK(ctx, cudaMemsetAsync(at<unsigned>(ws, L.cnt), 0, sizeof(unsigned) * (L.Pl > 1 ? L.Pl : 1), st));
    LAUNCH(ctx, 1, launch_pso_init(swarm_of(ws, L), L.P, L.Pl, L.p0, pso->v0, k0, k1, c0, L.nslots, st));
    if (L.mode != PIFCM_FIT_CHAINED)  // the shared state's centres
        CK(ctx, cudaMemcpyAsync(at<float>(ws, L.shc), c0, sizeof(float) * 4, cudaMemcpyDeviceToDevice, st));
    return PIFCM_OK;
}

int pifcm_pso_fitness_ptr(const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                          void *ws, double **fitness) {
    if (!fitness || !ws) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(nullptr, grid)) || (r = check_cfg(nullptr, cfg)) || (r = check_pso(nullptr, pso))) return r;
    *fitness = at<double>(ws, layout(grid, cfg, pso).fit);
    return PIFCM_OK;
}

int pifcm_pso_eval(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                   const float *x, void *ws, size_t ws_bytes, pifcm_stream stream) {
    Layout L;
    int r = pso_common(ctx, grid, cfg, pso, ws, ws_bytes, &L);
    if (r) return r;
    if (!x) return fail(ctx, PIFCM_EINVAL, "x is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    SwarmDev s = swarm_of(ws, L);
    float4 *slots = at<float4>(ws, L.slots);
    if (L.mode == PIFCM_FIT_CHAINED) {
        const int nblk = step_nblk(grid->nx, grid->ny, grid->nz, true, L.Pl);
        for (int b0 = 0; b0 < L.Pl; b0 += L.eb) {
            const int nb = L.Pl - b0 < L.eb ? L.Pl - b0 : L.eb;
            if (L.eb < L.Pl) LAUNCH(ctx, 1, launch_assign_batch(s, L.Pl, b0, nb, L.nslots, st));
            r = run_step(ctx, grid, cfg, x, slots, slots, s.cur + b0, s.nxt + b0, s.centers + 4 * b0,
                         s.pos + 2 * (L.p0 + b0), true, 0, nb, at<double>(ws, L.part) + (size_t)b0 * nblk * kNR,
                         s.fit + L.p0 + b0, nullptr, 0.f, s.hdr + kHStatus, s.hdr + kHStop, st, L.nslots,
                         at<unsigned>(ws, L.cnt) + b0);
            if (r) return r;
        }
        return PIFCM_OK;
    }
    // ANCHORED / LEADER: H, F of the shared state (ANCHORED: once per run, the
    // pass is skipped once hdr[kHHfValid] is set), then all particles' J
    float4 *hf = at<float4>(ws, L.hf);
    {
        StepArgs a{};
        a.x = x;
        a.nx = grid->nx; a.ny = grid->ny; a.nz = grid->nz; a.pitch = grid->pitch;
        a.nvox = L.nvox;
        a.U_in = slots; a.U_out = slots;
        a.in_idx = L.mode == PIFCM_FIT_LEADER ? s.cur : nullptr;  // ANCHORED: slot 0
        a.centers = at<float>(ws, L.shc);
        a.lam_xi = at<double>(ws, L.lamxi);
        a.stop = L.mode == PIFCM_FIT_ANCHORED ? s.hdr + kHHfValid : s.hdr + kHStop;
        a.m = cfg->m; a.inv_m1 = 1.0f / (cfg->m - 1.0f); a.q_mode = cfg->q_mode;
        set_shells(a, cfg);
        a.n_in_states = L.nslots;
        a.C = cfg->C;
        a.hf = hf;
        LAUNCH(ctx, 1, launch_step(a, cfg->C, true, 1, st));
        if (L.mode == PIFCM_FIT_ANCHORED) LAUNCH(ctx, 1, launch_set_hdr(s.hdr, kHHfValid, 1, st));
    }
    int nparts = 0;
    double *parts = at<double>(ws, L.part);
    LAUNCH(ctx, 1, launch_eval_shared(x, grid->nx, grid->ny, grid->nz, grid->pitch, hf, at<float>(ws, L.shc),
                                      s.pos + 2 * L.p0, L.Pl, cfg->C, cfg->m, parts, &nparts, st));
    LAUNCH(ctx, 1, launch_fit_sum(parts, nparts, L.Pl, s.fit + L.p0, s.hdr + kHStatus, st));
    return PIFCM_OK;
}

int pifcm_pso_trace(pifcm_ctx *ctx, double *f, double *pos, int32_t *gbest, int32_t max_gen) {
    if (!ctx) return PIFCM_EINVAL;
    const bool off = !f && !pos && !gbest;
    if (!off && (!f || !pos || !gbest || max_gen < 1))
        return fail(ctx, PIFCM_EINVAL, "pifcm_pso_trace: f, pos, gbest all non-NULL with max_gen >= 1, or all NULL");
    ctx->tr_f = f; ctx->tr_pos = pos; ctx->tr_gbest = gbest; ctx->tr_max = off ? 0 : max_gen;
    return PIFCM_OK;
}

int pifcm_pso_update(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                     const float *x, void *ws, size_t ws_bytes, pifcm_stream stream) {
    Layout L;
    int r = pso_common(ctx, grid, cfg, pso, ws, ws_bytes, &L);
    if (r) return r;
    if (L.mode != PIFCM_FIT_CHAINED && !x) return fail(ctx, PIFCM_EINVAL, "ANCHORED / LEADER updates need x");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    PsoUpdateArgs a{};
    a.s = swarm_of(ws, L);
    a.P = L.P; a.Pl = L.Pl; a.p0 = L.p0; a.ring_k = pso->ring_k; a.patience = pso->patience;
    a.nslots = L.nslots; a.tol = pso->tol; a.vmax = pso->vmax; a.mode = L.mode;
    a.batched = L.eb < L.Pl ? 1 : 0;
    a.key0 = (uint32_t)(pso->seed & 0xFFFFFFFFu); a.key1 = (uint32_t)(pso->seed >> 32);
    a.tr_f = ctx->tr_f; a.tr_pos = ctx->tr_pos; a.tr_gbest = ctx->tr_gbest; a.tr_max = ctx->tr_max;
    LAUNCH(ctx, 1, launch_pso_update(a, st));
    if (L.mode == PIFCM_FIT_CHAINED) return PIFCM_OK;
    // ANCHORED: on an improvement, the snapshot = one step from the start at the
    // gbest's evaluation position (slot 0 -> slot 1; skipped otherwise).
    // LEADER: S_{t+1} = one step from S_t at the gbest's evaluation position
    // (slot cur[0] -> nxt[0]); it becomes the shared state (and, on an
    // improvement, the pinned snapshot).
    SwarmDev s = a.s;
    float4 *slots = at<float4>(ws, L.slots);
    double *lamxi = at<double>(ws, L.lamxi);
    const bool anch = L.mode == PIFCM_FIT_ANCHORED;
    LAUNCH(ctx, 1, launch_mode_pre(s, at<float>(ws, L.shc), lamxi, L.mode, st));
    if (anch) {
        r = run_step(ctx, grid, cfg, x, slots, slots + L.nvox, nullptr, nullptr, s.gbest_c, lamxi, true, 0, 1,
                     at<double>(ws, L.part), nullptr, nullptr, 0.f, s.hdr + kHStatus, s.hdr + kHNotImproved, st, 1,
                     at<unsigned>(ws, L.cnt));
    } else {
        r = run_step(ctx, grid, cfg, x, slots, slots, s.cur, s.nxt, at<float>(ws, L.shc), lamxi, true, 0, 1,
                     at<double>(ws, L.part), nullptr, nullptr, 0.f, s.hdr + kHStatus, s.hdr + kHStop, st,
                     L.nslots, at<unsigned>(ws, L.cnt));
    }
    if (r) return r;
    if (!anch) LAUNCH(ctx, 1, launch_leader_post(s, at<float>(ws, L.shc), st));
    return PIFCM_OK;
}

int pifcm_pso_step(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                   const float *x, void *ws, size_t ws_bytes, pifcm_stream stream) {
    int r = pifcm_pso_eval(ctx, grid, cfg, pso, x, ws, ws_bytes, stream);
    if (r) return r;
    return pifcm_pso_update(ctx, grid, cfg, pso, x, ws, ws_bytes, stream);
}

int pifcm_pso_result_get(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                         const pifcm_pso_cfg *pso, void *ws, pifcm_pso_result *out, int32_t *stopped,
                         pifcm_stream stream) {
    if (!ctx || !out) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid)) || (r = check_cfg(ctx, cfg)) || (r = check_pso(ctx, pso))) return r;
    Layout L = layout(grid, cfg, pso);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int hdr[16];
    double dh[16];
    float gc[4];
    CK(ctx, cudaMemcpyAsync(hdr, at<int>(ws, L.hdr), sizeof hdr, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(dh, at<double>(ws, L.dhdr), sizeof dh, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(gc, at<float>(ws, L.gbc), sizeof gc, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    if (!hdr[kHInit]) return fail(ctx, PIFCM_ESTATE, "swarm not initialised (call pifcm_pso_init)");
    if (hdr[kHStatus]) return fail(ctx, hdr[kHStatus], "non-finite fitness during PSO");
    out->lambda = dh[kDGbestL];
    out->xi = dh[kDGbestX];
    out->J = dh[kDGbestJ];
    out->generations = hdr[kHGen];
    out->gbest_particle = hdr[kHGbest];
    for (int j = 0; j < 4; ++j) out->centers[j] = gc[j];
    if (stopped) *stopped = hdr[kHStop];
    return PIFCM_OK;
}

int pifcm_pso_gbest_state(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg,
                          const pifcm_pso_cfg *pso, void *ws, float *U_out, float *c_out, pifcm_stream stream) {
    if (!ctx || !U_out) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid)) || (r = check_cfg(ctx, cfg)) || (r = check_pso(ctx, pso))) return r;
    Layout L = layout(grid, cfg, pso);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int gs = -1;
    CK(ctx, cudaMemcpyAsync(&gs, at<int>(ws, L.hdr) + kHGbestSlot, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    if (gs < 0) return fail(ctx, PIFCM_ESTATE, "the gbest state is not held by this process");
    LAUNCH(ctx, 1, launch_gather_gbest(at<float4>(ws, L.slots), L.nvox, at<int>(ws, L.hdr), at<float>(ws, L.gbc),
                                       reinterpret_cast<float4 *>(U_out), c_out, st));
    return PIFCM_OK;
}

int pifcm_pso_run(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                  const float *x, const float *U0, const float *c0, void *ws, size_t ws_bytes,
                  pifcm_pso_result *out, pifcm_stream stream) {
    if (pso && !(pso->p_begin == 0 && pso->p_end == 0) && (pso->p_begin != 0 || pso->p_end != pso->P))
        return fail(ctx, PIFCM_EINVAL, "pifcm_pso_run is single-process: use eval/update for sharding");
    int r = pifcm_pso_init(ctx, grid, cfg, pso, U0, c0, ws, ws_bytes, stream);
    if (r) return r;
    const int check_every = 4;
    for (int gen = 0; gen < pso->max_gen; ++gen) {
        if ((r = pifcm_pso_step(ctx, grid, cfg, pso, x, ws, ws_bytes, stream))) return r;
        if (pso->patience > 0 && (gen + 1) % check_every == 0) {
            pifcm_pso_result tmp;
            int32_t stopped = 0;
            if ((r = pifcm_pso_result_get(ctx, grid, cfg, pso, ws, &tmp, &stopped, stream))) return r;
            if (stopped) break;
        }
    }
    if (out) return pifcm_pso_result_get(ctx, grid, cfg, pso, ws, out, nullptr, stream);
    return PIFCM_OK;
}

// ============================================================== ABI: pipeline parts
int pifcm_normalize(pifcm_ctx *ctx, const pifcm_grid *grid, const void *vol, int32_t dtype, float *x,
                    int64_t *hist, void *ws, size_t ws_bytes, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid))) return r;
    if (!vol || !x) return fail(ctx, PIFCM_EINVAL, "vol and x must be non-NULL");
    if (dtype != PIFCM_U8 && dtype != PIFCM_U16 && dtype != PIFCM_F32)
        return fail(ctx, PIFCM_EINVAL, "dtype %d unknown", dtype);
    if (!ws || ws_bytes < 256) return fail(ctx, PIFCM_ENOMEM, "normalize needs >= 256 bytes of workspace");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const long long n = (long long)grid->nx * grid->ny * grid->nz;
    unsigned int *mm = static_cast<unsigned int *>(ws);
    LAUNCH(ctx, 2, launch_minmax(vol, dtype, n, mm, st));
    LAUNCH(ctx, 1, launch_normalize(vol, dtype, grid->nx, grid->ny, grid->nz, grid->pitch, mm, x, st));
    if (hist) LAUNCH(ctx, 2, launch_hist(vol, dtype, n, mm, hist, st));
    return PIFCM_OK;
}

int pifcm_normalize_u8(pifcm_ctx *ctx, const pifcm_grid *grid, const uint8_t *vol, float *x, int64_t *hist,
                       void *ws, size_t ws_bytes, pifcm_stream stream) {
    return pifcm_normalize(ctx, grid, vol, PIFCM_U8, x, hist, ws, ws_bytes, stream);
}

int pifcm_gmm_init(pifcm_ctx *ctx, int32_t C, const int64_t *hist, float *c0, void *ws, size_t ws_bytes,
                   pifcm_stream stream) {
    (void)ws; (void)ws_bytes;
    if (!ctx) return PIFCM_EINVAL;
    if (C < 2 || C > kMaxC) return fail(ctx, PIFCM_EINVAL, "C = %d outside [2, 4]", C);
    if (!hist || !c0) return fail(ctx, PIFCM_EINVAL, "hist and c0 must be non-NULL");
    LAUNCH(ctx, 1, launch_gmm(hist, C, 100, c0, reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_value_hist(pifcm_ctx *ctx, const void *vol, int32_t dtype, int64_t n, int64_t *counts,
                     pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (dtype != PIFCM_U8 && dtype != PIFCM_U16)
        return fail(ctx, PIFCM_EINVAL, "value histogram of dtype %d: only PIFCM_U8 / PIFCM_U16", dtype);
    if (n < 0) return fail(ctx, PIFCM_EINVAL, "n = %lld < 0", (long long)n);
    if (n > 0 && (!vol || !counts)) return fail(ctx, PIFCM_EINVAL, "vol and counts must be non-NULL");
    if (n == 0) return PIFCM_OK;
    LAUNCH(ctx, 1, launch_value_hist(vol, dtype, n, counts, reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_fcm_hist_workspace_size(int32_t dtype, size_t *bytes) {
    if (!bytes || (dtype != PIFCM_U8 && dtype != PIFCM_U16)) return PIFCM_EINVAL;
    *bytes = fcm_hist_ws_bytes(dtype == PIFCM_U8 ? 256 : 65536);
    return PIFCM_OK;
}

int pifcm_fcm_hist(pifcm_ctx *ctx, const pifcm_ifcm_cfg *cfg, int32_t dtype, const uint32_t *mm,
                   const int64_t *counts, const float *c0, float *c_prev, float *c_out, double *stats, void *ws,
                   size_t ws_bytes, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if (!cfg) return fail(ctx, PIFCM_EINVAL, "cfg must be non-NULL");
    if ((r = check_cfg(ctx, cfg))) return r;
    if (dtype != PIFCM_U8 && dtype != PIFCM_U16)
        return fail(ctx, PIFCM_EINVAL, "value-histogram FCM of dtype %d: only PIFCM_U8 / PIFCM_U16", dtype);
    if (!mm || !counts || !c0 || !c_prev || !c_out || !stats)
        return fail(ctx, PIFCM_EINVAL, "mm, counts, c0, c_prev, c_out and stats must be non-NULL");
    const int nvals = dtype == PIFCM_U8 ? 256 : 65536;
    if ((r = check_ws(ctx, ws, ws_bytes, fcm_hist_ws_bytes(nvals)))) return r;
    FcmHistArgs fa = fcm_hist_args(ws, nvals);
    fa.counts = counts; fa.mm = mm; fa.c0 = c0; fa.max_iter = cfg->max_iter; fa.eps = cfg->eps;
    fa.m = cfg->m; fa.inv_m1 = 1.0f / (cfg->m - 1.0f); fa.c_prev = c_prev; fa.c_out = c_out; fa.stats = stats;
    fa.status = nullptr;
    LAUNCH(ctx, 1, launch_fcm_hist(fa, cfg->C, cfg->m == 2.0f, reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_fcm_memberships(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t C, float m, const float *x,
                          const float *c, float *U, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid))) return r;
    if (C < 2 || C > kMaxC) return fail(ctx, PIFCM_EINVAL, "C = %d outside [2, 4]", C);
    if (!(m > 1.0f)) return fail(ctx, PIFCM_EINVAL, "m = %g must be > 1", (double)m);
    if (!x || !c || !U) return fail(ctx, PIFCM_EINVAL, "x, c and U must be non-NULL");
    LAUNCH(ctx, 1, launch_fcm_memberships(x, grid->nx, grid->ny, grid->nz, (int)grid->pitch, c, C, m,
                                          reinterpret_cast<float4 *>(U), reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_incs(pifcm_ctx *ctx, const uint8_t *labels, const uint8_t *truth, int64_t n, int32_t C,
               const float *centers, int64_t *count, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (C < 2 || C > kMaxC) return fail(ctx, PIFCM_EINVAL, "C = %d outside [2, 4]", C);
    if (n < 0) return fail(ctx, PIFCM_EINVAL, "n = %lld < 0", (long long)n);
    if (!count || !centers || (n > 0 && (!labels || !truth)))
        return fail(ctx, PIFCM_EINVAL, "labels, truth, centers and count must be non-NULL");
    LAUNCH(ctx, 1, launch_incs(labels, truth, n, C, centers, count, reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_eq11(const double *incs, const double *secs, int32_t k, int32_t A, double alpha, double *J) {
    if (!incs || !secs || !J || k < 1 || A < 1 || !(alpha >= 0.0 && alpha <= 1.0)) return PIFCM_EINVAL;
    for (int a = 0; a < A; ++a) J[a] = 0.0;
    for (int i = 0; i < k; ++i) {
        const double *q = incs + (size_t)i * A, *t = secs + (size_t)i * A;
        double qlo = q[0], qhi = q[0], tlo = t[0], thi = t[0];
        for (int a = 1; a < A; ++a) {
            qlo = q[a] < qlo ? q[a] : qlo;
            qhi = q[a] > qhi ? q[a] : qhi;
            tlo = t[a] < tlo ? t[a] : tlo;
            thi = t[a] > thi ? t[a] : thi;
        }
        for (int a = 0; a < A; ++a)  // min-max normalisation per size; a constant row contributes 0 (R26)
            J[a] += alpha * (qhi > qlo ? (q[a] - qlo) / (qhi - qlo) : 0.0) +
                    (1.0 - alpha) * (thi > tlo ? (t[a] - tlo) / (thi - tlo) : 0.0);
    }
    for (int a = 0; a < A; ++a) J[a] /= (double)k;
    return PIFCM_OK;
}

int pifcm_argmax(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t C, const float *U, uint8_t *labels,
                 pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid))) return r;
    if (C < 2 || C > kMaxC) return fail(ctx, PIFCM_EINVAL, "C = %d outside [2, 4]", C);
    if (!U || !labels) return fail(ctx, PIFCM_EINVAL, "U and labels must be non-NULL");
    const long long n = (long long)grid->nx * grid->ny * grid->nz;
    LAUNCH(ctx, 1, launch_argmax(reinterpret_cast<const float4 *>(U), n, C, labels,
                                 reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

// ============================================================== ABI: pipeline
// Iterate state in slot `a` until eps / max_iter using slots a <-> b; returns
// the slot holding the result in *res and the iteration count in *iters.
static int run_until(pifcm_ctx *ctx, const pifcm_grid *g, const pifcm_ifcm_cfg *cfg, const float *x,
                     float4 *slots, long long nvox, int a, int b, float *centers, const double *lamxi,
                     bool stencil, bool fcm_first, double *partials, double *stats, int *status, unsigned *counters,
                     cudaStream_t st, int *res, int *iters, unsigned *gbar = nullptr) {
    CK(ctx, cudaMemsetAsync(stats, 0, sizeof(double) * 4, st));
    if (stencil && !fcm_first) {  // a 2D image: every iteration in one cooperative launch
        bool used = false;
        int r = run_2d_loop(ctx, g, cfg, x, slots + (long long)a * nvox, slots + (long long)b * nvox, centers, lamxi,
                            cfg->max_iter, partials, stats, status, counters, gbar, st, &used);
        if (r) return r;
        if (used) {
            double h[4];
            CK(ctx, cudaMemcpyAsync(h, stats, sizeof h, cudaMemcpyDeviceToHost, st));
            CK(ctx, cudaStreamSynchronize(st));
            const int done = (int)h[2];
            loop_timing_count(ctx, done, nvox);
            *iters = done;
            *res = (done % 2 == 1) ? b : a;
            return PIFCM_OK;
        }
    }
    int src = a, dst = b, t = 0;
    // the host checks the device's convergence flag every 16 iterations: once
    // converged the remaining launches return at once (a few us each), which
    // is cheaper than a host round trip per 4 iterations
    const int check_every = 16;
    for (t = 1; t <= cfg->max_iter; ++t) {
        int r = run_step(ctx, g, cfg, x, slots + (long long)src * nvox, slots + (long long)dst * nvox, nullptr,
                         nullptr, centers, lamxi, stencil, (fcm_first && t == 1) ? 1 : 0, 1, partials,
                         nullptr, stats, cfg->eps, status, nullptr, st, 1, counters,
                         /*canonical: identical to the z-slab sharded final IFCM*/ stencil);
        if (r) return r;
        const int tmp = src; src = dst; dst = tmp;
        if (t % check_every == 0 || t == cfg->max_iter) {
            double h[4];
            CK(ctx, cudaMemcpyAsync(h, stats, sizeof h, cudaMemcpyDeviceToHost, st));
            CK(ctx, cudaStreamSynchronize(st));
            if (h[3] != 0.0) {
                // converged at iteration h[2]; later launches were no-ops
                const int done = (int)h[2];
                *iters = done;
                *res = (done % 2 == 1) ? b : a;
                return PIFCM_OK;
            }
        }
    }
    *iters = cfg->max_iter;
    *res = (cfg->max_iter % 2 == 1) ? b : a;
    return PIFCM_OK;
}

int pifcm_segment(pifcm_ctx *ctx, const void *vol, int32_t dtype, int32_t nx, int32_t ny, int32_t nz,
                  const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso, int32_t z_slice, void *ws,
                  size_t ws_bytes, uint8_t *labels, float *U_out, pifcm_report *rep, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (dtype != PIFCM_U8 && dtype != PIFCM_U16 && dtype != PIFCM_F32)
        return fail(ctx, PIFCM_EINVAL, "dtype %d unknown", dtype);
    if (!vol || !labels) return fail(ctx, PIFCM_EINVAL, "vol and labels must be non-NULL");
    pifcm_grid g{nx, ny, nz, (nx + 3) / 4 * 4};
    Layout L;
    int r = pso_common(ctx, &g, cfg, pso, ws, ws_bytes, &L);
    if (r) return r;
    const bool sharded = ctx->comm.world > 1;
    if (sharded) {
        int a, b;
        pifcm::dist_range(pso->P, ctx->comm.world, ctx->comm.rank, &a, &b);
        if (pso->p_begin != a || pso->p_end != b)
            return fail(ctx, PIFCM_EINVAL, "rank %d of %d must evaluate particles [%d, %d) (pifcm_dist_range), not [%d, %d)",
                        ctx->comm.rank, ctx->comm.world, a, b, pso->p_begin, pso->p_end);
    } else if (!(pso->p_begin == 0 && pso->p_end == 0) && (pso->p_begin != 0 || pso->p_end != pso->P)) {
        return fail(ctx, PIFCM_EINVAL, "a particle sub-range needs a communicator (pifcm_ctx_dist)");
    }
    if (z_slice < -1 || z_slice >= nz) return fail(ctx, PIFCM_EINVAL, "z_slice %d out of range", z_slice);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CK(ctx, cudaSetDevice(ctx->device));
    cudaEvent_t *ev = ctx->ev;
    float *x = at<float>(ws, L.x);
    int64_t *hist = at<int64_t>(ws, L.hist);
    float *c0 = at<float>(ws, L.c0);
    float4 *slots = at<float4>(ws, L.slots);
    double *partials = at<double>(ws, L.part);
    double *stats = at<double>(ws, L.stats);
    double *lamxi = at<double>(ws, L.lamxi);
    SwarmDev s = swarm_of(ws, L);
    int *status = s.hdr + kHStatus;
    float *cent = s.centers;  // [Pl][4]; entry 0 reused by the FCM start and the final IFCM
    // NVTX ranges per phase (SURVEY 5 tracing; no cost without a profiler)
    struct Nvtx {
        bool open = false;
        void phase(const char *name) {
            if (open) nvtxRangePop();
            nvtxRangePushA(name);
            open = true;
        }
        ~Nvtx() { if (open) nvtxRangePop(); }
    } nvtx;
    nvtx.phase("pifcm: normalize (Alg. 2 step 1)");
    CK(ctx, cudaEventRecord(ev[0], st));
    // Alg. 2 step 1: normalise (+ histogram for the GMM start)

    unsigned int *mm = at<unsigned int>(ws, L.mm);
    LAUNCH(ctx, 2, launch_minmax(vol, dtype, L.nvox, mm, st));
    LAUNCH(ctx, 1, launch_normalize(vol, dtype, nx, ny, nz, g.pitch, mm, x, st));
    LAUNCH(ctx, 2, launch_hist(vol, dtype, L.nvox, mm, hist, st));
    CK(ctx, cudaEventRecord(ev[1], st));
    nvtx.phase("pifcm: GMM + FCM start (Alg. 1 step 2)");
    // Alg. 1 step 2: GMM centres, then FCM (lambda = xi = 0) until eps
    LAUNCH(ctx, 1, launch_gmm(hist, cfg->C, 100, c0, st));
    float cinit[4];
    CK(ctx, cudaMemcpyAsync(cinit, c0, sizeof cinit, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(cent, c0, sizeof(float) * 4, cudaMemcpyDeviceToDevice, st));
    CK(ctx, cudaMemsetAsync(lamxi, 0, sizeof(double) * 2, st));
    CK(ctx, cudaMemsetAsync(s.hdr, 0, sizeof(int) * 16, st));
    CK(ctx, cudaMemsetAsync(at<unsigned>(ws, L.cnt), 0, sizeof(unsigned) * (L.Pl > 1 ? L.Pl : 1), st));
    int fcm_slot = 0, fcm_iters = 0;
    const bool vh = dtype != PIFCM_F32;
    if (vh) {
        // quantised input: the FCM loop on the value histogram (R24), then
        // the memberships of every voxel once, into slot 0 (the PSO start)
        const int nvals = dtype == PIFCM_U8 ? 256 : 65536;
        int64_t *vcnt = at<int64_t>(ws, L.vcnt);
        CK(ctx, cudaMemsetAsync(vcnt, 0, sizeof(int64_t) * nvals, st));
        LAUNCH(ctx, 1, launch_value_hist(vol, dtype, L.nvox, vcnt, st));
        FcmHistArgs fa = fcm_hist_args(at<void>(ws, L.fhws), nvals);
        fa.counts = vcnt; fa.mm = mm; fa.c0 = c0; fa.max_iter = cfg->max_iter; fa.eps = cfg->eps;
        fa.m = cfg->m; fa.inv_m1 = 1.0f / (cfg->m - 1.0f); fa.c_prev = at<float>(ws, L.cprev);
        fa.c_out = cent; fa.stats = at<double>(ws, L.fstats); fa.status = status;
        LAUNCH(ctx, 1, launch_fcm_hist(fa, cfg->C, cfg->m == 2.0f, st));
        LAUNCH(ctx, 1, launch_fcm_memberships(x, nx, ny, nz, g.pitch, fa.c_prev, cfg->C, cfg->m, slots, st));
    } else {
        if ((r = run_until(ctx, &g, cfg, x, slots, L.nvox, 1, 0, cent, lamxi, false, true, partials, stats, status,
                           at<unsigned>(ws, L.cnt), st, &fcm_slot, &fcm_iters)))
            return r;
        // keep the FCM result in slot 0 (the PSO start slot)
        if (fcm_slot != 0)
            CK(ctx, cudaMemcpyAsync(slots, slots + (long long)fcm_slot * L.nvox, sizeof(float4) * (size_t)L.nvox,
                                    cudaMemcpyDeviceToDevice, st));
    }
    CK(ctx, cudaMemcpyAsync(c0, cent, sizeof(float) * 4, cudaMemcpyDeviceToDevice, st));
    CK(ctx, cudaEventRecord(ev[2], st));
    nvtx.phase("pifcm: PSO (Alg. 1 steps 3-10)");
    // Alg. 1 steps 3-10: PSO (c0 now holds the FCM centres for pso_init)
    pifcm_pso_result pres;
    if (!sharded) {
        if ((r = pifcm_pso_run(ctx, &g, cfg, pso, x, reinterpret_cast<float *>(slots), c0, ws, ws_bytes, &pres,
                               stream)))
            return r;
    } else {
        // particle-sharded generations: local evaluation, fitness all-gather,
        // the identical update on every rank (Alg. 1 steps 4-9)
        if ((r = pifcm_pso_init(ctx, &g, cfg, pso, reinterpret_cast<float *>(slots), c0, ws, ws_bytes, stream)))
            return r;
        for (int gen = 0; gen < pso->max_gen; ++gen) {
            if ((r = pifcm_pso_eval(ctx, &g, cfg, pso, x, ws, ws_bytes, stream))) return r;
            std::string err;
            if ((r = pifcm::comm_allgather_fitness(ctx->comm, s.fit, pso->P, st, err)))
                return fail(ctx, r, "fitness all-gather: %s", err.c_str());
            if ((r = pifcm_pso_update(ctx, &g, cfg, pso, x, ws, ws_bytes, stream))) return r;
            if (pso->patience > 0 && (gen + 1) % 4 == 0) {
                int32_t stopped = 0;
                if ((r = pifcm_pso_result_get(ctx, &g, cfg, pso, ws, &pres, &stopped, stream))) return r;
                if (stopped) break;
            }
        }
        if ((r = pifcm_pso_result_get(ctx, &g, cfg, pso, ws, &pres, nullptr, stream))) return r;
    }
    CK(ctx, cudaEventRecord(ev[3], st));
    nvtx.phase("pifcm: final IFCM (Alg. 1 step 11)");
    // Alg. 1 step 11: final IFCM from the gbest state at (lambda*, xi*)
    int gs = -1;
    CK(ctx, cudaMemcpyAsync(&gs, s.hdr + kHGbestSlot, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    if (sharded && L.mode == PIFCM_FIT_CHAINED) {
        // Alg. 1 step 10 across ranks: the owner's gbest state (slot + centres)
        // into slot 0 of every rank
        int owner = 0;
        for (int q = 0; q < ctx->comm.world; ++q) {
            int a, b;
            pifcm::dist_range(pso->P, ctx->comm.world, q, &a, &b);
            if (pres.gbest_particle >= a && pres.gbest_particle < b) owner = q;
        }
        if (ctx->comm.rank == owner) {
            if (gs < 0) return fail(ctx, PIFCM_ESTATE, "gbest owner holds no gbest state");
            if (gs != 0)
                CK(ctx, cudaMemcpyAsync(slots, slots + (long long)gs * L.nvox, sizeof(float4) * (size_t)L.nvox,
                                        cudaMemcpyDeviceToDevice, st));
        }
        std::string err;
        if ((r = pifcm::comm_broadcast(ctx->comm, slots, sizeof(float4) * (size_t)L.nvox, owner, st, err)) ||
            (r = pifcm::comm_broadcast(ctx->comm, s.gbest_c, sizeof(float) * 4, owner, st, err)))
            return fail(ctx, r, "gbest broadcast: %s", err.c_str());
        gs = 0;
    }
    if (gs < 0) return fail(ctx, PIFCM_ESTATE, "no gbest state after PSO");
    const int other = (gs == 0) ? 1 : 0;
    CK(ctx, cudaMemcpyAsync(cent, s.gbest_c, sizeof(float) * 4, cudaMemcpyDeviceToDevice, st));
    LAUNCH(ctx, 1, launch_set_lamxi(lamxi, s.dhdr, st));
    const bool zero = (pres.lambda == 0.0 && pres.xi == 0.0);
    int fin_slot = gs, fin_iters = 0;
    if ((r = run_until(ctx, &g, cfg, x, slots, L.nvox, gs, other, cent, lamxi, !zero, false, partials, stats, status,
                       at<unsigned>(ws, L.cnt), st, &fin_slot, &fin_iters, at<unsigned>(ws, L.gbar))))
        return r;
    CK(ctx, cudaEventRecord(ev[4], st));
    nvtx.phase("pifcm: defuzzify");
    // defuzzify (+ optional U copy)
    const float4 *Ufin = slots + (long long)fin_slot * L.nvox;
    if (z_slice < 0) {
        LAUNCH(ctx, 1, launch_argmax(Ufin, L.nvox, cfg->C, labels, st));
    } else {
        const long long plane = (long long)nx * ny;
        LAUNCH(ctx, 1, launch_argmax(Ufin + (long long)z_slice * plane, plane, cfg->C, labels, st));
    }
    if (U_out)
        CK(ctx, cudaMemcpyAsync(U_out, Ufin, sizeof(float4) * (size_t)L.nvox, cudaMemcpyDeviceToDevice, st));
    CK(ctx, cudaEventRecord(ev[5], st));
    float cfin[4];
    int stat = 0;
    CK(ctx, cudaMemcpyAsync(cfin, cent, sizeof cfin, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(&stat, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    double fst[4] = {0.0, 0.0, 0.0, 0.0};
    if (vh) CK(ctx, cudaMemcpyAsync(fst, at<double>(ws, L.fstats), sizeof fst, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    CK(ctx, cudaGetLastError());
    if (vh) fcm_iters = (int)fst[2];
    if (stat) return fail(ctx, stat, "non-finite cost during the pipeline");
    if (rep) {
        memset(rep, 0, sizeof *rep);
        rep->pso = pres;
        rep->fcm_iters = fcm_iters;
        rep->final_iters = fin_iters;
        for (int j = 0; j < 4; ++j) { rep->centers[j] = cfin[j]; rep->c_init[j] = cinit[j]; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[0], ev[1]); rep->t_norm = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[1], ev[2]); rep->t_init = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[2], ev[3]); rep->t_pso = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[3], ev[4]); rep->t_final = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[0], ev[5]); rep->t_total = ms * 1e-3;
    }
    return PIFCM_OK;
}

int pifcm_segment_host(pifcm_ctx *ctx, const uint8_t *vol_host, int32_t nx, int32_t ny, int32_t nz,
                       const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes,
                       uint8_t *labels_host, pifcm_report *rep, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (!vol_host || !labels_host) return fail(ctx, PIFCM_EINVAL, "host buffers must be non-NULL");
    pifcm_grid g{nx, ny, nz, (nx + 3) / 4 * 4};
    Layout L;
    int r = pso_common(ctx, &g, cfg, pso, ws, ws_bytes, &L);
    if (r) return r;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint8_t *dvol = at<uint8_t>(ws, L.vol), *dlab = at<uint8_t>(ws, L.lab);
    CK(ctx, cudaMemcpyAsync(dvol, vol_host, (size_t)L.nvox, cudaMemcpyHostToDevice, st));
    if ((r = pifcm_segment(ctx, dvol, PIFCM_U8, nx, ny, nz, cfg, pso, -1, ws, ws_bytes, dlab, nullptr, rep, stream)))
        return r;
    CK(ctx, cudaMemcpyAsync(labels_host, dlab, (size_t)L.nvox, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    return PIFCM_OK;
}

// ============================================================== ABI: z-slab
// The slice mode's single-plane slab (R25): its halo planes are the fixed
// neighbour rows, refilled by pifcm_segment_slice itself.
static bool slab_is_slice(const pifcm_grid *g) { return g && g->nz == 1; }

// H = halo planes per side of the slab arrays (= cfg->v, the neighbourhood
// radius in z); slice: the single-plane slab of the slice mode, whose halo
// planes are the fixed neighbour rows, not a neighbour rank's planes.
static int check_slab(pifcm_ctx *ctx, const pifcm_grid *g, int H = 1, bool slice = false) {
    if (!g) return fail(ctx, PIFCM_EINVAL, "grid is NULL");
    if (g->nx < 1 || g->ny < 1 || g->nz < 1) return fail(ctx, PIFCM_EINVAL, "grid dims must be >= 1");
    if (g->pitch < g->nx || g->pitch % 4 != 0) return fail(ctx, PIFCM_EALIGN, "pitch must be >= nx and % 4 == 0");
    if (g->nz_total < 1) return fail(ctx, PIFCM_EINVAL, "slab calls need nz_total >= 1");
    if (g->z0 < 0 || g->z0 + g->nz > g->nz_total)
        return fail(ctx, PIFCM_EINVAL, "slab [%d, %d) outside [0, %d)", g->z0, g->z0 + g->nz, g->nz_total);
    // (a single-plane slab -- the slice mode, R25 -- is one chunk at any z0)
    const int tz = slab_tz(g->nx, g->ny, g->nz_total);
    if (g->nz > 1 && g->z0 % tz != 0)
        return fail(ctx, PIFCM_EINVAL, "slab z0 = %d is not a multiple of %d", g->z0, tz);
    if (g->nz > 1 && g->z0 + g->nz != g->nz_total && g->nz % tz != 0)
        return fail(ctx, PIFCM_EINVAL, "a slab other than the last must hold a multiple of %d planes", tz);
    if ((long long)g->nx * g->ny * (g->nz + 2 * H) >= (1LL << 31)) return fail(ctx, PIFCM_EINVAL, "slab too large");
    // a slab's neighbours take their H halo planes from its own planes only
    // (a thinner slab is allowed where the other side is outside the volume)
    if (!slice && g->nz < H && g->z0 > 0 && g->z0 + g->nz < g->nz_total)
        return fail(ctx, PIFCM_EINVAL, "an interior slab needs >= %d planes for v = %d", H, H);
    return PIFCM_OK;
}

int pifcm_slab_records(const pifcm_grid *grid, int32_t *nrec) {
    if (!nrec) return PIFCM_EINVAL;
    int r;
    if ((r = check_slab(nullptr, grid))) return r;
    const int tz = slab_tz(grid->nx, grid->ny, grid->nz_total);
    *nrec = ((grid->nx + kTX - 1) / kTX) * ((grid->ny + kTY - 1) / kTY) * ((grid->nz + tz - 1) / tz);
    return PIFCM_OK;
}

int pifcm_slab_chunk(int32_t nx, int32_t ny, int32_t nz_total, int32_t *tz) {
    if (!tz || nx < 1 || ny < 1 || nz_total < 1) return PIFCM_EINVAL;
    *tz = slab_tz(nx, ny, nz_total);
    return PIFCM_OK;
}

int pifcm_slab_step(pifcm_ctx *ctx, const pifcm_grid *grid, const pifcm_ifcm_cfg *cfg, const float *x,
                    const float *U_in, float *U_out, const float *centers, const double *lam_xi, int32_t P,
                    const double *stats, double *records, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if (!cfg) return fail(ctx, PIFCM_EINVAL, "cfg is NULL");
    if ((r = check_cfg(ctx, cfg)) || (r = check_slab(ctx, grid, cfg->v, slab_is_slice(grid)))) return r;
    const int H = cfg->v;  // halo planes per side (Eq. 9 radius in z)
    if (P < 1 || P > 65535) return fail(ctx, PIFCM_EINVAL, "P = %d outside [1, 65535]", P);
    if (!x || !U_in || !U_out || !centers || !lam_xi || !records)
        return fail(ctx, PIFCM_EINVAL, "x, U_in, U_out, centers, lam_xi and records must be non-NULL");
    if (U_in == U_out) return fail(ctx, PIFCM_EINVAL, "U_in and U_out must not alias");
    StepArgs a{};
    a.x = x;
    a.nx = grid->nx; a.ny = grid->ny; a.nz = grid->nz + 2 * H; a.pitch = grid->pitch;
    a.nvox = (long long)grid->nx * grid->ny * (grid->nz + 2 * H);
    a.z_lo = H; a.nz_t = grid->nz; a.goff = grid->z0 - H; a.nz_g = grid->nz_total;
    set_shells(a, cfg);
    a.U_in = reinterpret_cast<const float4 *>(U_in); a.U_out = reinterpret_cast<float4 *>(U_out);
    a.centers = const_cast<float *>(centers); a.lam_xi = lam_xi; a.partials = records;
    a.stats = stats;
    a.m = cfg->m; a.inv_m1 = 1.0f / (cfg->m - 1.0f); a.q_mode = cfg->q_mode;
    a.n_in_states = P;
    a.want_du = 1;
    a.counters = nullptr;  // records are combined across ranks by pifcm_slab_finalize
    a.C = cfg->C;
    return timed_step(ctx, a, cfg->C, true, P, (long long)grid->nx * grid->ny * grid->nz,
                      reinterpret_cast<cudaStream_t>(stream));
}

int pifcm_slab_finalize(pifcm_ctx *ctx, int32_t C, int32_t P, int32_t world, int32_t nrec, const int32_t *counts,
                        const double *records, float *centers, double *stats, double *fitness, float eps,
                        pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (C < 2 || C > kMaxC || P < 1 || world < 1 || world > 64 || nrec < 1 || !records || !centers)
        return fail(ctx, PIFCM_EINVAL, "invalid slab finalize arguments");
    LAUNCH(ctx, 1, launch_slab_finalize(C, P, world, nrec, counts, records, centers, stats, fitness, eps, nullptr,
                                        reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_slab_halo_v(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t v, int32_t P, int32_t op, float *U,
                      float *buf, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if (v < 1 || v > kMaxV) return fail(ctx, PIFCM_EINVAL, "v = %d outside [1, %d]", v, kMaxV);
    if ((r = check_slab(ctx, grid, v))) return r;
    if (P < 1 || op < 0 || op > 3 || !U) return fail(ctx, PIFCM_EINVAL, "invalid halo arguments");
    const int H = v;
    const long long plane = (long long)grid->nx * grid->ny;
    const long long state = plane * (grid->nz + 2 * H);
    float4 *U4 = reinterpret_cast<float4 *>(U), *B4 = reinterpret_cast<float4 *>(buf);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (op <= 1) {  // the first / last H local planes -> buf [P][H planes]
        if (!buf) return fail(ctx, PIFCM_EINVAL, "pack needs a buffer");
        const long long src_plane = op == 0 ? H : grid->nz;
        LAUNCH(ctx, 1, launch_halo_copy(U4 + src_plane * plane, state, B4, H * plane, H * plane, P, false, st));
    } else {  // buf -> the lower / upper H halo planes (zeros outside the volume)
        const long long dst_plane = op == 2 ? 0 : grid->nz + H;
        const bool outside = op == 2 ? grid->z0 == 0 : grid->z0 + grid->nz == grid->nz_total;
        if (!outside && !buf) return fail(ctx, PIFCM_EINVAL, "unpack of an interior halo needs a buffer");
        LAUNCH(ctx, 1, launch_halo_copy(B4, H * plane, U4 + dst_plane * plane, state, H * plane, P, outside, st));
    }
    return PIFCM_OK;
}

int pifcm_slab_halo(pifcm_ctx *ctx, const pifcm_grid *grid, int32_t P, int32_t op, float *U, float *buf,
                    pifcm_stream stream) {
    return pifcm_slab_halo_v(ctx, grid, 1, P, op, U, buf, stream);
}


// ============================================================== ABI: pipeline parts for slabs
int pifcm_minmax_u8(pifcm_ctx *ctx, const uint8_t *vol, int64_t n, uint32_t *mm, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (!vol || !mm || n < 1) return fail(ctx, PIFCM_EINVAL, "vol, mm non-NULL and n >= 1 required");
    LAUNCH(ctx, 2, launch_minmax_u8(vol, n, reinterpret_cast<unsigned int *>(mm),
                                    reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_normalize_u8_range(pifcm_ctx *ctx, const pifcm_grid *grid, const uint8_t *vol, const uint32_t *mm,
                             float *x, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if ((r = check_grid(ctx, grid))) return r;
    if (!vol || !mm || !x) return fail(ctx, PIFCM_EINVAL, "vol, mm and x must be non-NULL");
    LAUNCH(ctx, 1, launch_normalize_u8(vol, grid->nx, grid->ny, grid->nz, grid->pitch,
                                       reinterpret_cast<const unsigned int *>(mm), x,
                                       reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_hist_u8(pifcm_ctx *ctx, const uint8_t *vol, int64_t n, const uint32_t *mm, int64_t *hist,
                  pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    if (!vol || !mm || !hist || n < 1) return fail(ctx, PIFCM_EINVAL, "vol, mm, hist non-NULL and n >= 1 required");
    LAUNCH(ctx, 2, launch_hist_u8(vol, n, reinterpret_cast<const unsigned int *>(mm), hist,
                                  reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

// ============================================================== ABI: PSO over z-slabs
// The swarm of a slab rank lives in a pifcm workspace laid out for the slab's
// arrays (nz + 2v planes with the halos); every rank holds all particles.
static pifcm_grid plain_of(const pifcm_grid *s, int H) {
    return pifcm_grid{s->nx, s->ny, s->nz + 2 * H, s->pitch, 0, 0};
}

static int slab_pso_common(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                           const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes, Layout *L, pifcm_grid *pg) {
    int r;
    if (!cfg) return fail(ctx, PIFCM_EINVAL, "cfg is NULL");
    if ((r = check_cfg(ctx, cfg)) || (r = check_slab(ctx, slab, cfg->v, slab_is_slice(slab))) ||
        (r = check_pso(ctx, pso)))
        return r;
    if (!(pso->p_begin == 0 && pso->p_end == 0) && (pso->p_begin != 0 || pso->p_end != pso->P))
        return fail(ctx, PIFCM_EINVAL, "slab ranks hold every particle (p_begin = p_end = 0)");
    if (pso->fitness_mode != PIFCM_FIT_CHAINED) return fail(ctx, PIFCM_EINVAL, "slab PSO: CHAINED fitness only");
    *pg = plain_of(slab, cfg->v);
    *L = layout(pg, cfg, pso);
    if (ctx) CK(ctx, cudaSetDevice(ctx->device));
    return ws ? check_ws(ctx, ws, ws_bytes, L->total) : PIFCM_OK;
}

int pifcm_slab_workspace_size(const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                              size_t *bytes) {
    if (!bytes) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(nullptr, slab, cfg, pso, nullptr, 0, &L, &pg);
    if (r) return r;
    *bytes = L.total;
    return PIFCM_OK;
}

int pifcm_slab_pso_init(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                        const float *U0, const float *c0, void *ws, size_t ws_bytes, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, ws, ws_bytes, &L, &pg);
    if (r) return r;
    return pifcm_pso_init(ctx, &pg, cfg, pso, U0, c0, ws, ws_bytes, stream);
}

int pifcm_slab_pso_halo(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                        void *ws, size_t ws_bytes, int32_t op, float *buf, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, ws, ws_bytes, &L, &pg);
    if (r) return r;
    if (op < 0 || op > 3) return fail(ctx, PIFCM_EINVAL, "halo op %d outside [0, 3]", op);
    const int H = cfg->v;
    const long long plane = (long long)slab->nx * slab->ny, hp = H * plane;
    SwarmDev s = swarm_of(ws, L);
    float4 *slots = at<float4>(ws, L.slots), *B4 = reinterpret_cast<float4 *>(buf);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (op <= 1) {
        if (!buf) return fail(ctx, PIFCM_EINVAL, "pack needs a buffer");
        const long long src_plane = op == 0 ? H : slab->nz;
        LAUNCH(ctx, 1, launch_halo_copy(slots + src_plane * plane, L.nvox, B4, hp, hp, L.Pl, false, st, s.cur,
                                        nullptr));
    } else {
        const long long dst_plane = op == 2 ? 0 : slab->nz + H;
        const bool outside = op == 2 ? slab->z0 == 0 : slab->z0 + slab->nz == slab->nz_total;
        if (!outside && !buf) return fail(ctx, PIFCM_EINVAL, "unpack of an interior halo needs a buffer");
        LAUNCH(ctx, 1, launch_halo_copy(B4, hp, slots + dst_plane * plane, L.nvox, hp, L.Pl, outside, st,
                                        nullptr, s.cur));
    }
    return PIFCM_OK;
}

int pifcm_slab_pso_eval(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso,
                        const float *x, void *ws, size_t ws_bytes, double *records, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, ws, ws_bytes, &L, &pg);
    if (r) return r;
    if (!x || !records) return fail(ctx, PIFCM_EINVAL, "x and records must be non-NULL");
    SwarmDev s = swarm_of(ws, L);
    float4 *slots = at<float4>(ws, L.slots);
    StepArgs a{};
    a.x = x;
    const int H = cfg->v;
    a.nx = slab->nx; a.ny = slab->ny; a.nz = slab->nz + 2 * H; a.pitch = slab->pitch;
    a.nvox = L.nvox;
    a.z_lo = H; a.nz_t = slab->nz; a.goff = slab->z0 - H; a.nz_g = slab->nz_total;
    set_shells(a, cfg);
    a.U_in = slots; a.U_out = slots;
    a.stop = s.hdr + kHStop;
    a.m = cfg->m; a.inv_m1 = 1.0f / (cfg->m - 1.0f); a.q_mode = cfg->q_mode;
    a.n_in_states = L.nslots;
    a.counters = nullptr;  // records are combined across ranks by pifcm_slab_pso_finalize
    a.C = cfg->C;
    int nrec = 0;
    if ((r = pifcm_slab_records(slab, &nrec))) return fail(ctx, r, "invalid slab grid");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    for (int b0 = 0; b0 < L.Pl; b0 += L.eb) {  // batches of eval_batch states (see pifcm_pso_eval)
        const int nb = L.Pl - b0 < L.eb ? L.Pl - b0 : L.eb;
        if (L.eb < L.Pl) LAUNCH(ctx, 1, launch_assign_batch(s, L.Pl, b0, nb, L.nslots, st));
        a.in_idx = s.cur + b0; a.out_idx = s.nxt + b0;
        a.centers = s.centers + 4 * b0; a.lam_xi = s.pos + 2 * b0;
        a.partials = records + (size_t)b0 * nrec * kNR;
        if ((r = timed_step(ctx, a, cfg->C, true, nb, (long long)slab->nx * slab->ny * slab->nz, st))) return r;
    }
    return PIFCM_OK;
}

int pifcm_slab_pso_finalize(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                            const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes, int32_t world, int32_t nrec,
                            const int32_t *counts, const double *records, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, ws, ws_bytes, &L, &pg);
    if (r) return r;
    if (world < 1 || world > 64 || nrec < 1 || !records) return fail(ctx, PIFCM_EINVAL, "invalid records");
    SwarmDev s = swarm_of(ws, L);
    LAUNCH(ctx, 1, launch_slab_finalize(cfg->C, L.Pl, world, nrec, counts, records, s.centers, nullptr, s.fit, 0.f,
                                        s.hdr + kHStatus, reinterpret_cast<cudaStream_t>(stream)));
    return PIFCM_OK;
}

int pifcm_slab_pso_update(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                          const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, ws, ws_bytes, &L, &pg);
    if (r) return r;
    return pifcm_pso_update(ctx, &pg, cfg, pso, nullptr, ws, ws_bytes, stream);
}

int pifcm_slab_pso_result_get(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                              const pifcm_pso_cfg *pso, void *ws, pifcm_pso_result *out, int32_t *stopped,
                              pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, nullptr, 0, &L, &pg);
    if (r) return r;
    return pifcm_pso_result_get(ctx, &pg, cfg, pso, ws, out, stopped, stream);
}

int pifcm_slab_pso_gbest_state(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg,
                               const pifcm_pso_cfg *pso, void *ws, float *U_out, float *c_out, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    Layout L;
    pifcm_grid pg;
    int r = slab_pso_common(ctx, slab, cfg, pso, nullptr, 0, &L, &pg);
    if (r) return r;
    return pifcm_pso_gbest_state(ctx, &pg, cfg, pso, ws, U_out, c_out, stream);
}


// ============================================================== ABI: peer memory
int pifcm_peer_alloc(pifcm_ctx *ctx, size_t bytes, void **ptr) {
    if (!ctx || !ptr || bytes == 0) return PIFCM_EINVAL;
    CK(ctx, cudaSetDevice(ctx->device));
    CK(ctx, cudaMalloc(ptr, bytes));
    CK(ctx, cudaMemset(*ptr, 0, bytes));
    return PIFCM_OK;
}
int pifcm_peer_free(pifcm_ctx *ctx, void *ptr) {
    if (!ctx) return PIFCM_EINVAL;
    CK(ctx, cudaSetDevice(ctx->device));
    CK(ctx, cudaFree(ptr));
    return PIFCM_OK;
}
int pifcm_peer_handle(pifcm_ctx *ctx, void *ptr, uint8_t *handle) {
    if (!ctx || !ptr || !handle) return PIFCM_EINVAL;
    cudaIpcMemHandle_t h;
    CK(ctx, cudaSetDevice(ctx->device));
    CK(ctx, cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof h == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle, &h, sizeof h);
    return PIFCM_OK;
}
int pifcm_peer_open(pifcm_ctx *ctx, const uint8_t *handle, void **ptr) {
    if (!ctx || !ptr || !handle) return PIFCM_EINVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    CK(ctx, cudaSetDevice(ctx->device));
    CK(ctx, cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return PIFCM_OK;
}
int pifcm_peer_close(pifcm_ctx *ctx, void *ptr) {
    if (!ctx) return PIFCM_EINVAL;
    CK(ctx, cudaSetDevice(ctx->device));
    CK(ctx, cudaIpcCloseMemHandle(ptr));
    return PIFCM_OK;
}

int pifcm_slab_p2p_run(pifcm_ctx *ctx, const pifcm_grid *slab, const pifcm_ifcm_cfg *cfg, const float *x,
                       const pifcm_peers *peers, int32_t P, const int32_t *counts, int32_t nrec_max,
                       float *centers, const double *lam_xi, double *stats, double *rec_local, int32_t iters,
                       uint32_t *epoch, int32_t *cur, int32_t *iters_done, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    int r;
    if (!cfg) return fail(ctx, PIFCM_EINVAL, "cfg is NULL");
    if ((r = check_cfg(ctx, cfg)) || (r = check_slab(ctx, slab, cfg->v))) return r;
    const int H = cfg->v;
    if (!peers || !x || !centers || !lam_xi || !stats || !rec_local || !epoch || !cur || !iters_done)
        return fail(ctx, PIFCM_EINVAL, "NULL argument");
    const int world = peers->world, rank = peers->rank;
    if (world < 1 || world > PIFCM_MAX_PEERS || rank < 0 || rank >= world || P < 1 || iters < 1 ||
        (*cur != 0 && *cur != 1) || peers->nz[rank] != slab->nz)
        return fail(ctx, PIFCM_EINVAL, "invalid peer description");
    int32_t nrec = 0;
    if ((r = pifcm_slab_records(slab, &nrec))) return fail(ctx, r, "slab records");
    if (nrec > nrec_max) return fail(ctx, PIFCM_EINVAL, "nrec_max %d < this slab's %d records", nrec_max, nrec);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CK(ctx, cudaSetDevice(ctx->device));
    const long long plane = (long long)slab->nx * slab->ny;
    unsigned *myflags = peers->flags[rank];
    int *status = reinterpret_cast<int *>(myflags + world + 1);
    CK(ctx, cudaMemsetAsync(stats, 0, sizeof(double) * 4 * P, st));
    auto put = [&](int buf, bool records, unsigned e) -> int {
        P2PPut a{};
        a.src = reinterpret_cast<const float4 *>(peers->U[buf][rank]);
        a.plane = plane;
        a.H = H;
        a.state = plane * (slab->nz + 2 * H);
        a.nz = slab->nz;
        a.P = P;
        if (rank > 0) {  // our first H planes -> rank-1's upper halo
            a.lo_dst = reinterpret_cast<float4 *>(peers->U[buf][rank - 1]) + (long long)(peers->nz[rank - 1] + H) * plane;
            a.lo_state = plane * (peers->nz[rank - 1] + 2 * H);
        }
        if (rank < world - 1) {  // our last H planes -> rank+1's lower halo
            a.hi_dst = reinterpret_cast<float4 *>(peers->U[buf][rank + 1]);
            a.hi_state = plane * (peers->nz[rank + 1] + 2 * H);
        }
        a.rec_src = records ? rec_local : nullptr;
        a.nrec = nrec; a.nrec_max = nrec_max; a.world = world; a.rank = rank;
        for (int w = 0; w < world; ++w) {
            a.rec_dst[w] = peers->rec[e & 1u][w];
            a.flags[w] = peers->flags[w];
        }
        a.counter = myflags + world;
        a.epoch = e;
        LAUNCH(ctx, 1, launch_p2p_put(a, st));
        LAUNCH(ctx, 1, launch_p2p_wait(myflags, world, e, status, st));
        return PIFCM_OK;
    };
    unsigned e = *epoch;
    int c = *cur;
    // halos of the starting states
    if ((r = put(c, false, ++e))) return r;
    int t = 0;
    const int check_every = 16;
    for (t = 1; t <= iters; ++t) {
        if ((r = pifcm_slab_step(ctx, slab, cfg, x, peers->U[c][rank], peers->U[1 - c][rank], centers, lam_xi, P,
                                 stats, rec_local, stream)))
            return r;
        if ((r = put(1 - c, true, ++e))) return r;
        LAUNCH(ctx, 1, launch_slab_finalize(cfg->C, P, world, nrec_max, counts, peers->rec[e & 1u][rank], centers,
                                            stats, nullptr, cfg->eps, nullptr, st));
        c = 1 - c;
        if (t % check_every == 0 || t == iters) {
            std::vector<double> h(4 * (size_t)P);
            int hs = 0;
            CK(ctx, cudaMemcpyAsync(h.data(), stats, sizeof(double) * 4 * P, cudaMemcpyDeviceToHost, st));
            CK(ctx, cudaMemcpyAsync(&hs, status, sizeof hs, cudaMemcpyDeviceToHost, st));
            CK(ctx, cudaStreamSynchronize(st));
            if (hs) return fail(ctx, PIFCM_ECUDA, "peer barrier timed out at epoch %u", e);
            bool all = cfg->eps > 0.f;
            for (int p = 0; p < P && all; ++p) all = h[4 * p + 3] != 0.0;
            if (all) break;
        }
    }
    *epoch = e;
    *cur = c;
    *iters_done = t > iters ? iters : t;
    return PIFCM_OK;
}

// ============================================================== ABI: slice mode
// The literal slice mode (R25; Alg. 1 with its input z):
// slice z is segmented with its 3D neighbourhood; the neighbour planes
// z - v .. z - 1, z + 1 .. z + v (Eq. 9 radius v in z) carry the FCM start's
// memberships at its centres c1, fixed.  The slice is a single-plane slab
// (pifcm_slab_* calls, nz = 1, z0 = z): its state slots hold the 2v halo
// planes, refilled with the fixed rows before every evaluation; the final
// IFCM iterates the slab step + finalisation.
namespace {
struct SliceLayout {
    Layout L;           // the slab PSO workspace (offset 0)
    size_t xs, hlo, hhi, A, B, rec, mm, hist, vcnt, fhws, c0, cprev, c1, cent, lamxi, stats, fstats, status, total;
    long long plane;
    int nrec;
};
SliceLayout slice_layout(const pifcm_grid *sg, const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso) {
    SliceLayout S{};
    const int H = cfg->v;  // neighbour planes per side (Eq. 9 radius in z)
    const pifcm_grid pg{sg->nx, sg->ny, 1 + 2 * H, sg->pitch, 0, 0};
    S.L = layout(&pg, cfg, pso);
    S.plane = (long long)sg->nx * sg->ny;
    const int tz = slab_tz(sg->nx, sg->ny, sg->nz_total);
    S.nrec = ((sg->nx + kTX - 1) / kTX) * ((sg->ny + kTY - 1) / kTY) * ((1 + tz - 1) / tz);
    size_t o = S.L.total;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
    S.xs = take(sizeof(float) * (1 + 2 * H) * (size_t)sg->ny * sg->pitch);
    S.hlo = take(sizeof(float4) * H * (size_t)S.plane);
    S.hhi = take(sizeof(float4) * H * (size_t)S.plane);
    S.A = take(sizeof(float4) * (1 + 2 * H) * (size_t)S.plane);
    S.B = take(sizeof(float4) * (1 + 2 * H) * (size_t)S.plane);
    S.rec = take(sizeof(double) * kNR * (size_t)S.nrec * (pso->P > 1 ? pso->P : 1));
    S.mm = take(sizeof(unsigned) * 2);
    S.hist = take(sizeof(int64_t) * 256);
    S.vcnt = take(sizeof(int64_t) * 256);
    S.fhws = take(fcm_hist_ws_bytes(256));
    S.c0 = take(sizeof(float) * 4);
    S.cprev = take(sizeof(float) * 4);
    S.c1 = take(sizeof(float) * 4);
    S.cent = take(sizeof(float) * 4);
    S.lamxi = take(sizeof(double) * 2);
    S.stats = take(sizeof(double) * 4);
    S.fstats = take(sizeof(double) * 4);
    S.status = take(sizeof(int) * 4);
    S.total = o;
    return S;
}
int slice_check(pifcm_ctx *ctx, int32_t nx, int32_t ny, int32_t nz, int32_t z, const pifcm_ifcm_cfg *cfg,
                const pifcm_pso_cfg *pso, pifcm_grid *sg) {
    if (nx < 1 || ny < 1 || nz < 1) return fail(ctx, PIFCM_EINVAL, "grid dims must be >= 1");
    if (z < 0 || z >= nz) return fail(ctx, PIFCM_EINVAL, "slice z = %d outside [0, %d)", z, nz);
    *sg = pifcm_grid{nx, ny, 1, (nx + 3) / 4 * 4, z, nz};
    int r;
    if ((r = check_slab(ctx, sg)) || (r = check_cfg(ctx, cfg)) || (r = check_pso(ctx, pso))) return r;
    if (pso->fitness_mode != PIFCM_FIT_CHAINED) return fail(ctx, PIFCM_EINVAL, "slice mode: CHAINED fitness");
    if (!(pso->p_begin == 0 && pso->p_end == 0) && (pso->p_begin != 0 || pso->p_end != pso->P))
        return fail(ctx, PIFCM_EINVAL, "slice mode is single-process");
    return PIFCM_OK;
}
}  // namespace

int pifcm_segment_slice_workspace_size(int32_t nx, int32_t ny, int32_t nz, int32_t z, const pifcm_ifcm_cfg *cfg,
                                       const pifcm_pso_cfg *pso, size_t *bytes) {
    if (!bytes) return PIFCM_EINVAL;
    pifcm_grid sg;
    int r = slice_check(nullptr, nx, ny, nz, z, cfg, pso, &sg);
    if (r) return r;
    *bytes = slice_layout(&sg, cfg, pso).total;
    return PIFCM_OK;
}

int pifcm_segment_slice(pifcm_ctx *ctx, const uint8_t *vol, int32_t nx, int32_t ny, int32_t nz, int32_t z,
                        const pifcm_ifcm_cfg *cfg, const pifcm_pso_cfg *pso, void *ws, size_t ws_bytes,
                        uint8_t *labels, float *U_out, pifcm_report *rep, pifcm_stream stream) {
    if (!ctx) return PIFCM_EINVAL;
    pifcm_grid sg;
    int r = slice_check(ctx, nx, ny, nz, z, cfg, pso, &sg);
    if (r) return r;
    if (!vol || !labels) return fail(ctx, PIFCM_EINVAL, "vol and labels must be non-NULL");
    const SliceLayout S = slice_layout(&sg, cfg, pso);
    if ((r = check_ws(ctx, ws, ws_bytes, S.total))) return r;
    CK(ctx, cudaSetDevice(ctx->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaEvent_t *ev = ctx->ev;
    const long long plane = S.plane, N = plane * nz;
    const int pitch = sg.pitch;
    float *xs = at<float>(ws, S.xs);
    float4 *hlo = at<float4>(ws, S.hlo), *hhi = at<float4>(ws, S.hhi), *A = at<float4>(ws, S.A),
           *B = at<float4>(ws, S.B);
    unsigned *mm = at<unsigned>(ws, S.mm);
    int *status = at<int>(ws, S.status);
    const int H = cfg->v;  // neighbour planes per side
    const long long hp = H * plane;
    CK(ctx, cudaEventRecord(ev[0], st));
    CK(ctx, cudaMemsetAsync(status, 0, sizeof(int) * 4, st));
    // Alg. 2 step 1: the volume's range; x of planes z - H .. z + H (0 outside)
    LAUNCH(ctx, 2, launch_minmax(vol, PIFCM_U8, N, mm, st));
    for (int k = 0; k < 1 + 2 * H; ++k) {
        const int gz = z - H + k;
        float *xk = xs + (size_t)k * ny * pitch;
        if (gz < 0 || gz >= nz)
            CK(ctx, cudaMemsetAsync(xk, 0, sizeof(float) * (size_t)ny * pitch, st));
        else
            LAUNCH(ctx, 1, launch_normalize(vol + (long long)gz * plane, PIFCM_U8, nx, ny, 1, pitch, mm, xk, st));
    }
    // Alg. 1 steps 1-2: R15 histogram of the slice on the volume's levels, GMM,
    // FCM on the slice (value histogram, R24)
    int64_t *hist = at<int64_t>(ws, S.hist), *vcnt = at<int64_t>(ws, S.vcnt);
    LAUNCH(ctx, 2, launch_hist(vol + (long long)z * plane, PIFCM_U8, plane, mm, hist, st));
    float *c0 = at<float>(ws, S.c0), *cprev = at<float>(ws, S.cprev), *c1 = at<float>(ws, S.c1),
          *cent = at<float>(ws, S.cent);
    LAUNCH(ctx, 1, launch_gmm(hist, cfg->C, 100, c0, st));
    float cinit[4];
    CK(ctx, cudaMemcpyAsync(cinit, c0, sizeof cinit, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaEventRecord(ev[1], st));
    CK(ctx, cudaMemsetAsync(vcnt, 0, sizeof(int64_t) * 256, st));
    LAUNCH(ctx, 1, launch_value_hist(vol + (long long)z * plane, PIFCM_U8, plane, vcnt, st));
    FcmHistArgs fa = fcm_hist_args(at<void>(ws, S.fhws), 256);
    fa.counts = vcnt; fa.mm = mm; fa.c0 = c0; fa.max_iter = cfg->max_iter; fa.eps = cfg->eps;
    fa.m = cfg->m; fa.inv_m1 = 1.0f / (cfg->m - 1.0f); fa.c_prev = cprev; fa.c_out = c1;
    fa.stats = at<double>(ws, S.fstats); fa.status = status;
    LAUNCH(ctx, 1, launch_fcm_hist(fa, cfg->C, cfg->m == 2.0f, st));
    // the start state: slice rows from the FCM's last iteration, the fixed
    // neighbour rows = Eq. 2 at c1 (zero outside the volume)
    LAUNCH(ctx, 1, launch_fcm_memberships(xs + (size_t)H * ny * pitch, nx, ny, 1, pitch, cprev, cfg->C, cfg->m,
                                          A + hp, st));
    for (int k = 0; k < 1 + 2 * H; ++k) {
        if (k == H) continue;
        const int gz = z - H + k;
        float4 *dst = k < H ? hlo + (long long)k * plane : hhi + (long long)(k - H - 1) * plane;
        if (gz < 0 || gz >= nz) CK(ctx, cudaMemsetAsync(dst, 0, sizeof(float4) * plane, st));
        else LAUNCH(ctx, 1, launch_fcm_memberships(xs + (size_t)k * ny * pitch, nx, ny, 1, pitch, c1, cfg->C,
                                                   cfg->m, dst, st));
    }
    CK(ctx, cudaMemcpyAsync(A, hlo, sizeof(float4) * hp, cudaMemcpyDeviceToDevice, st));
    CK(ctx, cudaMemcpyAsync(A + hp + plane, hhi, sizeof(float4) * hp, cudaMemcpyDeviceToDevice, st));
    CK(ctx, cudaEventRecord(ev[2], st));
    // Alg. 1 steps 3-10: CHAINED PSO over the slice
    const Layout &L = S.L;
    double *rec = at<double>(ws, S.rec);
    if ((r = pifcm_slab_pso_init(ctx, &sg, cfg, pso, reinterpret_cast<float *>(A), c1, ws, L.total, stream)))
        return r;
    SwarmDev s = swarm_of(ws, L);
    float4 *slots = at<float4>(ws, L.slots);
    for (int gen = 0; gen < pso->max_gen; ++gen) {
        // the neighbour planes of every current state (new states carry stale halos)
        LAUNCH(ctx, 1, launch_halo_copy(hlo, 0, slots, L.nvox, hp, L.Pl, false, st, nullptr, s.cur));
        LAUNCH(ctx, 1, launch_halo_copy(hhi, 0, slots + hp + plane, L.nvox, hp, L.Pl, false, st, nullptr, s.cur));
        if ((r = pifcm_slab_pso_eval(ctx, &sg, cfg, pso, xs, ws, L.total, rec, stream))) return r;
        if ((r = pifcm_slab_pso_finalize(ctx, &sg, cfg, pso, ws, L.total, 1, S.nrec, nullptr, rec, stream)))
            return r;
        if ((r = pifcm_slab_pso_update(ctx, &sg, cfg, pso, ws, L.total, stream))) return r;
        if (pso->patience > 0 && (gen + 1) % 4 == 0) {
            int32_t stopped = 0;
            pifcm_pso_result tmp;
            if ((r = pifcm_slab_pso_result_get(ctx, &sg, cfg, pso, ws, &tmp, &stopped, stream))) return r;
            if (stopped) break;
        }
    }
    pifcm_pso_result pres;
    if ((r = pifcm_slab_pso_result_get(ctx, &sg, cfg, pso, ws, &pres, nullptr, stream))) return r;
    CK(ctx, cudaEventRecord(ev[3], st));
    // Alg. 1 step 11: final IFCM of the slice from the gbest state
    if ((r = pifcm_slab_pso_gbest_state(ctx, &sg, cfg, pso, ws, reinterpret_cast<float *>(A), cent, stream)))
        return r;
    for (float4 *T : {A, B}) {
        CK(ctx, cudaMemcpyAsync(T, hlo, sizeof(float4) * hp, cudaMemcpyDeviceToDevice, st));
        CK(ctx, cudaMemcpyAsync(T + hp + plane, hhi, sizeof(float4) * hp, cudaMemcpyDeviceToDevice, st));
    }
    double *lamxi = at<double>(ws, S.lamxi), *stats = at<double>(ws, S.stats);
    LAUNCH(ctx, 1, launch_set_lamxi(lamxi, s.dhdr, st));
    CK(ctx, cudaMemsetAsync(stats, 0, sizeof(double) * 4, st));
    int fin_iters = cfg->max_iter;
    for (int t = 1; t <= cfg->max_iter; ++t) {
        const float4 *src = (t % 2 == 1) ? A : B;
        float4 *dst = (t % 2 == 1) ? B : A;
        if ((r = pifcm_slab_step(ctx, &sg, cfg, xs, reinterpret_cast<const float *>(src),
                                 reinterpret_cast<float *>(dst), cent, lamxi, 1, stats, rec, stream)))
            return r;
        LAUNCH(ctx, 1, launch_slab_finalize(cfg->C, 1, 1, S.nrec, nullptr, rec, cent, stats, nullptr, cfg->eps,
                                            status, st));
        if (t % 16 == 0 || t == cfg->max_iter) {
            double h[4];
            CK(ctx, cudaMemcpyAsync(h, stats, sizeof h, cudaMemcpyDeviceToHost, st));
            CK(ctx, cudaStreamSynchronize(st));
            if (h[3] != 0.0) { fin_iters = (int)h[2]; break; }
        }
    }
    const float4 *Ufin = (fin_iters % 2 == 1) ? B : A;
    CK(ctx, cudaEventRecord(ev[4], st));
    LAUNCH(ctx, 1, launch_argmax(Ufin + hp, plane, cfg->C, labels, st));
    if (U_out)
        CK(ctx, cudaMemcpyAsync(U_out, Ufin + hp, sizeof(float4) * (size_t)plane, cudaMemcpyDeviceToDevice, st));
    CK(ctx, cudaEventRecord(ev[5], st));
    float cfin[4];
    int stat = 0;
    double fst[4];
    CK(ctx, cudaMemcpyAsync(cfin, cent, sizeof cfin, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(&stat, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(fst, at<double>(ws, S.fstats), sizeof fst, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    CK(ctx, cudaGetLastError());
    if (stat) return fail(ctx, stat, "non-finite cost during the slice pipeline");
    if (rep) {
        memset(rep, 0, sizeof *rep);
        rep->pso = pres;
        rep->fcm_iters = (int)fst[2];
        rep->final_iters = fin_iters;
        for (int j = 0; j < 4; ++j) { rep->centers[j] = cfin[j]; rep->c_init[j] = cinit[j]; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[0], ev[1]); rep->t_norm = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[1], ev[2]); rep->t_init = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[2], ev[3]); rep->t_pso = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[3], ev[4]); rep->t_final = ms * 1e-3;
        cudaEventElapsedTime(&ms, ev[0], ev[5]); rep->t_total = ms * 1e-3;
    }
    return PIFCM_OK;
}

}  // extern "C"
