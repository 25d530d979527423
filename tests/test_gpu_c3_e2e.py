"""End-to-end parity at the bench's exact configuration -- BASELINE.json's
north_star Target, "full PSO-tuned 3DPIFCM segmentation of a 181x217x181
volume matching the oracle": C3 (BrainWeb-shaped phantom, 9 % noise), C = 4,
m = 2, P = 32 particles, 30 generations, PSO seed 12345, final IFCM until
max|du| < 1e-5 or 100 iterations (Alg. 1; Alg. 2).

Three comparisons, all on the GPU's own trajectory through the C ABI:
  1. the swarm: identical evaluation positions, gbest sequence and
     (lambda*, xi*) on both sides (PSO arithmetic is fp64 on both sides, so
     equal comparisons give bit-identical trajectories), and per-generation
     fitness of every particle (the product path's pifcm_segment, recorded by
     pifcm_pso_trace) within 1e-5 relative of the oracle's own pso_run for the
     first EARLY generations -- after that the chained map at lambda = xi = 1
     amplifies rounding (tests/test_oracle_chaos.py), so the per-generation
     differences are recorded, and parity deep in the run is (2);
  2. same-state parity (north_star: memberships 1e-4 absolute, centres 1e-4
     relative) of one IFCM step from GPU states deep in the run -- particles
     replayed on the GPU to generations 0, 15 and 29 (each replay's cost is
     checked bit for bit against the trace, so it is the bench's state), and
     the final IFCM's iterations 0, 50 and 99 from the gbest snapshot;
  3. the final labels against the oracle's pipeline (orc_segment_u8's steps),
     agreement reported and required >= 99.9 % (north_star).
The oracle side is ~10 min of fp64 on the host cores (the whole C3 PSO)."""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

P, GENS, SEED, C = 32, 30, 12345, 4
U_TOL, C_TOL, F_TOL = 1e-4, 1e-4, 1e-5
EARLY = 3  # generations compared trajectory to trajectory (see the fitness assertion)
DEV = "cuda:0"


@pytest.fixture(scope="module")
def ctx():
    from paper_2002_01981_b200 import Context
    return Context(0)


def _gpu_start(ctx, vt, cfg):
    """pifcm_segment's Alg. 1 step 2 through the ABI parts: x, GMM c0, the FCM
    start on the value histogram (R24) -> (x, U1, c1, c0)."""
    mm = torch.zeros(64, dtype=torch.int32, device=DEV)
    x, hist = ctx.normalize(vt, mm=mm)
    c0 = ctx.gmm_init(hist, C)
    counts = ctx.value_hist(vt)
    c_prev, c1, _ = ctx.fcm_hist(counts, mm, c0, cfg)
    nz, ny, nx = vt.shape
    U1 = ctx.fcm_memberships(x, c_prev, C, cfg.m, nx)
    return x, U1, c1, c0


def _step(ctx, x, U, c, lam_xi, cfg, nx, canonical=False):
    """One pifcm_iterate step of one state -> (U_new [N,4], c_new [4], stats [4])."""
    N = U.shape[0]
    Uo = torch.empty_like(U)
    cen = c.clone().view(1, 4)
    lx = torch.tensor([lam_xi], dtype=torch.float64, device=DEV)
    st = torch.zeros((1, 4), dtype=torch.float64, device=DEV)
    ctx.iterate(x, U.view(1, N, 4), Uo.view(1, N, 4), cen, lx, cfg, iters=1, stats=st, nx=nx,
                canonical=canonical)
    return Uo, cen.view(4), st.view(4)


def _same_state(orc, xn, U, c, lam, xi, Ug, cg):
    """Oracle step from the GPU's fp32 state widened to fp64 vs the GPU's step."""
    Un = U.cpu().numpy()[:, :C].astype(np.float64)
    cn = c.cpu().numpy()[:C].astype(np.float64)
    Uo, co, Jo, _ = orc.ifcm_step(xn, Un, cn, lam, xi)
    du = float(np.abs(Ug.cpu().numpy()[:, :C] - Uo).max())
    dc = float(np.max(np.abs(cg.cpu().numpy()[:C] - co) / np.abs(co)))
    return du, dc, Jo


def test_c3_bench_config_end_to_end(ctx, orc):
    from inputs import config_volume
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    from paper_2002_01981_b200.api import _grid

    vol, _ = config_volume("C3")
    nz, ny, nx = vol.shape
    vt = torch.as_tensor(vol, device=DEV)
    cfg = IfcmConfig(C=C)
    pso = PsoConfig(P=P, max_gen=GENS, patience=0, seed=SEED)
    rec = {"config": "C3 181x217x181, C=4, m=2, P=32, 30 generations, seed 12345, eps 1e-5, <=100 final"}

    # ---- the product path (what bench.py times), with the swarm recorded
    tf = torch.zeros((GENS, P), dtype=torch.float64, device=DEV)
    tp = torch.zeros((GENS, P, 2), dtype=torch.float64, device=DEV)
    tg = torch.zeros(GENS, dtype=torch.int32, device=DEV)
    ctx.pso_trace(tf, tp, tg)
    labels_p, _, rep = ctx.segment(vt, cfg, pso, want_U=True)
    ctx.pso_trace(None)
    tf, tp, tg = tf.cpu().numpy(), tp.cpu().numpy(), tg.cpu().numpy()
    labels_p = labels_p.cpu().numpy().reshape(nz, ny, nx)

    # ---- the same pipeline through the ABI parts (replays need its states)
    x, U1, c1, c0 = _gpu_start(ctx, vt, cfg)
    xn = x[..., :nx].cpu().numpy().astype(np.float64)
    g = _grid(nx, ny, nz)
    ws = ctx.workspace(nx, ny, nz, cfg, pso)
    tf2 = torch.zeros((GENS, P), dtype=torch.float64, device=DEV)
    tp2 = torch.zeros((GENS, P, 2), dtype=torch.float64, device=DEV)
    tg2 = torch.zeros(GENS, dtype=torch.int32, device=DEV)
    ctx.pso_trace(tf2, tp2, tg2)
    ctx.pso_init(g, cfg, pso, U1, c1, ws)
    for _ in range(GENS):
        ctx.pso_step(g, cfg, pso, x, ws)
    ctx.pso_trace(None)
    summ, _ = ctx.pso_result(g, cfg, pso, ws)
    # the parts reproduce the product path bit for bit
    assert np.array_equal(tf2.cpu().numpy(), tf) and np.array_equal(tp2.cpu().numpy(), tp)
    assert np.array_equal(tg2.cpu().numpy(), tg)
    assert (summ.lam, summ.xi) == (rep["lambda"], rep["xi"])

    # ---- 2a. same-state parity deep in the swarm: replay particles to gen t
    same = []
    for p in (0, 17, P - 1):
        U, c = U1.clone(), c1.clone()
        for t in range(GENS):
            lam, xi = tp[t, p]
            Un, cn, st = _step(ctx, x, U, c, (lam, xi), cfg, nx)
            # the replay is the bench's state: its cost is the traced fitness, bit for bit
            assert st[0].item() == tf[t, p], (p, t, st[0].item(), tf[t, p])
            if t in (0, 15, GENS - 1):
                du, dc, _ = _same_state(orc, xn, U, c, lam, xi, Un, cn)
                same.append({"particle": p, "generation": t, "lam": lam, "xi": xi, "max_du": du,
                             "max_dc_rel": dc})
                assert du < U_TOL and dc < C_TOL, same[-1]
            U, c = Un, cn
    rec["same_state_swarm"] = same

    # ---- 2b. the final IFCM from the gbest snapshot, same-state at 0 / 50 / 99
    N = nx * ny * nz
    Ug = torch.empty((N, 4), dtype=torch.float32, device=DEV)
    cgb = torch.zeros(4, dtype=torch.float32, device=DEV)
    ctx.pso_gbest_state(g, cfg, pso, ws, Ug, cgb)
    lam_s, xi_s = summ.lam, summ.xi
    U, c = Ug, cgb
    fin = []
    it = 0
    for it in range(1, cfg.max_iter + 1):
        Un, cn, st = _step(ctx, x, U, c, (lam_s, xi_s), cfg, nx, canonical=True)
        if it - 1 in (0, 50, 99):
            du, dc, _ = _same_state(orc, xn, U, c, lam_s, xi_s, Un, cn)
            fin.append({"iteration": it - 1, "max_du": du, "max_dc_rel": dc})
            assert du < U_TOL and dc < C_TOL, fin[-1]
        U, c = Un, cn
        if st[1].item() < cfg.eps:
            break
    rec["same_state_final"] = fin
    labels_m = ctx.argmax(U, nx, ny, nz, C).cpu().numpy().reshape(nz, ny, nx)
    assert it == rep["final_iters"], (it, rep["final_iters"])
    assert np.array_equal(labels_m, labels_p)

    # ---- 1. + 3. the oracle's own pipeline (orc_segment_u8's steps)
    x64 = orc.normalize_u8(vol)
    c0o = orc.gmm_init(orc.histogram_u8(vol), C)
    U1o, c1o, fcm_it = orc.fcm_run(x64, c0o)
    r = orc.pso_run(x64, U1o, c1o, P=P, max_gen=GENS, seed=SEED)
    Uf, cf, fin_it, _ = orc.ifcm_run(x64, r.U, r.c, r.lam, r.xi)
    labels_o = orc.argmax(Uf).reshape(nz, ny, nx)

    rel = np.abs(tf - r.trace_f) / np.abs(r.trace_f)
    rec["fitness_max_rel_by_generation"] = rel.max(axis=1).tolist()
    rec["fitness_median_rel_by_generation"] = np.median(rel, axis=1).tolist()
    gb = r.trace_gbest
    rec["gbest_fitness_rel_by_generation"] = [float(rel[t, gb[t]]) for t in range(GENS)]
    rec["positions_identical"] = bool(np.array_equal(tp, r.trace_pos))
    rec["gbest_identical"] = bool(np.array_equal(tg, r.trace_gbest))
    rec["lambda_xi"] = {"gpu": [rep["lambda"], rep["xi"]], "oracle": [r.lam, r.xi]}
    rec["final_iters"] = {"gpu": rep["final_iters"], "oracle": fin_it}
    rec["centers"] = {"gpu": list(rep["centers"]), "oracle": cf.tolist()}
    agree = float((labels_p == labels_o).mean())
    rec["label_agreement"] = agree
    out = os.environ.get("PIFCM_E2E_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(rec, fh, indent=1)
    print(json.dumps(rec))
    assert rec["positions_identical"] and rec["gbest_identical"]
    assert (rep["lambda"], rep["xi"]) == (r.lam, r.xi)
    # fitness within 1e-5 while the swarm's states are still rounding-close;
    # later the chained map at lambda = xi = 1 amplifies fp32-vs-fp64
    # rounding (tests/test_oracle_chaos.py shows the oracle itself diverging
    # this way from an fp32-rounded start), so deep generations are compared
    # from the same state above instead
    assert rel[:EARLY].max() <= F_TOL, rel[:EARLY].max(axis=1)
    assert agree >= 0.999, agree
