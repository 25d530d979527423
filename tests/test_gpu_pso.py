"""GPU parity of the device PSO (Alg. 1 steps 3-10) and of the whole pipeline
(pifcm_segment) against the fp64 oracle, through the C ABI."""
import ctypes as ct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2002_01981_b200 import Context
    return Context(0)


def _small_case(C=3, shape=(10, 24, 28), seed=4):
    from inputs import cube_phantom, add_noise_u8
    nz, ny, nx = shape
    img, lab = cube_phantom(nx, ny, nz, (0.1, 0.5, 0.9) if C == 3 else (0.1, 0.35, 0.65, 0.9))
    vol = add_noise_u8(img, 7.0, seed)
    return vol, lab


def _setup_swarm(ctx, orc, P, seed, C=3, shape=(10, 24, 28)):
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig, to_aos, to_pitched_x
    from paper_2002_01981_b200.api import _grid
    vol, _ = _small_case(C=C, shape=shape)
    x = (vol.astype(np.float32) / 255.0)
    Uf, cf, _ = orc.fcm_run(x, np.linspace(0.1, 0.9, C))
    U0 = Uf.astype(np.float32)
    c0 = cf.astype(np.float32)
    nz, ny, nx = x.shape
    cfg = IfcmConfig(C=C)
    pso = PsoConfig(P=P, max_gen=50, patience=0, seed=seed)
    dev = torch.device("cuda:0")
    xt = to_pitched_x(x, dev)
    Ut = to_aos(U0, dev)
    c4 = torch.zeros(4, device=dev)
    c4[:C] = torch.as_tensor(c0)
    ws = ctx.workspace(nx, ny, nz, cfg, pso)
    g = _grid(nx, ny, nz)
    ctx.pso_init(g, cfg, pso, Ut, c4, ws)
    return x, U0, c0, cfg, pso, xt, Ut, ws, g


def test_pso_update_bit_exact(ctx, orc):
    """The device PSO bookkeeping (Alg. 1 steps 5-8) is bit-identical to the
    oracle's for the same fitness values: fitness injected into the device
    fitness vector from a fixed function of the oracle's positions."""
    P, seed, G = 7, 4242, 25
    x, U0, c0, cfg, pso, xt, Ut, ws, g = _setup_swarm(ctx, orc, P, seed)
    fit = ctx.pso_fitness(g, cfg, pso, ws)
    pos, vel = orc.pso_init(P, seed)
    pbf = np.full(P, np.inf)
    pbx = pos.copy()
    gb = -1
    for t in range(G):
        f = (pos[:, 0] - 0.3) ** 2 + (pos[:, 1] - 0.7) ** 2 + 0.01 * np.sin(7 * pos[:, 0] * pos[:, 1])
        eval_pos = pos.copy()
        fit.copy_(torch.as_tensor(f, device=fit.device))
        ctx.pso_update(g, cfg, pso, ws)
        gb, imp = orc.pso_update(f, pos, vel, pbf, pbx, gb, t, seed)
        summ, _ = ctx.pso_result(g, cfg, pso, ws)
        assert summ.gbest_particle == gb
        assert summ.J == pbf[gb]
        if imp:
            assert summ.lam == eval_pos[gb, 0] and summ.xi == eval_pos[gb, 1]
    assert summ.generations == G


def test_pso_gbest_tie_keeps_incumbent(ctx, orc):
    """R13 on the device: an exact fp64 tie with the incumbent gbest leaves
    the gbest (and so the owner of the pinned snapshot) unchanged; a strictly
    better pbest takes it (tests/test_oracle_pins_init.py's worked example)."""
    P, seed = 4, 5
    x, U0, c0, cfg, pso, xt, Ut, ws, g = _setup_swarm(ctx, orc, P, seed)
    fit = ctx.pso_fitness(g, cfg, pso, ws)
    pos, vel = orc.pso_init(P, seed)
    pbf = np.full(P, np.inf)
    pbx = pos.copy()
    gb = -1
    for t, (f, want) in enumerate((([5.0, 4.0, 2.0, 3.0], 2), ([2.0, 9.0, 9.0, 9.0], 2),
                                   ([1.0, 9.0, 9.0, 9.0], 0))):
        fit.copy_(torch.as_tensor(f, dtype=torch.float64, device=fit.device))
        ctx.pso_update(g, cfg, pso, ws)
        gb, _ = orc.pso_update(np.array(f), pos, vel, pbf, pbx, gb, t, seed)
        summ, _ = ctx.pso_result(g, cfg, pso, ws)
        assert summ.gbest_particle == gb == want
        assert summ.J == pbf[gb]


def test_pso_eval_parity(ctx, orc):
    """Generations 0 and 1 of the CHAINED fitness (one IFCM step per particle
    from its own state) within 1e-5 / 1e-4 of the oracle's."""
    P, seed = 6, 777
    x, U0, c0, cfg, pso, xt, Ut, ws, g = _setup_swarm(ctx, orc, P, seed)
    fit = ctx.pso_fitness(g, cfg, pso, ws)
    r = orc.pso_run(x, U0, c0, P=P, max_gen=2, seed=seed)
    for gen, tol in ((0, 1e-5), (1, 1e-4)):
        ctx.pso_eval(g, cfg, pso, xt, ws)
        f = fit.cpu().numpy()
        assert np.allclose(f, r.trace_f[gen], rtol=tol, atol=0), (gen, f, r.trace_f[gen])
        ctx.pso_update(g, cfg, pso, ws)
        summ, _ = ctx.pso_result(g, cfg, pso, ws)
        assert summ.gbest_particle == r.trace_gbest[gen]
    assert abs(summ.lam - r.lam) == 0 and abs(summ.xi - r.xi) == 0
    assert abs(summ.J - r.J) <= 1e-4 * r.J
    assert np.allclose(summ.centers, r.c, rtol=1e-4)
    # the gbest state (the U its evaluation produced), Alg. 1 step 10
    Ug = torch.empty_like(Ut)
    cg = torch.empty(4, device=Ut.device)
    ctx.pso_gbest_state(g, cfg, pso, ws, Ug, cg)
    assert np.abs(Ug.cpu().numpy()[:, :3] - r.U).max() < 1e-4


def test_pso_run_early_stop(ctx, orc):
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig, to_aos, to_pitched_x
    vol, _ = _small_case(C=2, shape=(6, 16, 16))
    x = vol.astype(np.float32) / 255.0
    Uf, cf, _ = orc.fcm_run(x, np.array([0.2, 0.8]))
    dev = torch.device("cuda:0")
    cfg = IfcmConfig(C=2)
    pso = PsoConfig(P=4, max_gen=40, patience=3, tol=1e-4, seed=1)
    c4 = torch.zeros(4, device=dev)
    c4[:2] = torch.as_tensor(cf.astype(np.float32))
    s = ctx.pso_run(to_pitched_x(x, dev), to_aos(Uf, dev), c4, cfg, pso, nx=16)
    r = orc.pso_run(x, Uf.astype(np.float32), cf.astype(np.float32), P=4, max_gen=40, seed=1,
                    patience=3, tol=1e-4)
    assert r.generations < 40
    # the device checks the stop flag every 4 generations; generations counted agree
    assert s.generations == r.generations
    assert abs(s.lam - r.lam) < 1e-12 and abs(s.xi - r.xi) < 1e-12


@pytest.mark.parametrize("C,shape,P,G,seed", [(3, (10, 24, 28), 4, 2, 99), (4, (1, 64, 64), 6, 2, 5),
                                              (2, (5, 9, 40), 3, 3, 99), (4, (6, 33, 35), 5, 2, 1)])
def test_segment_parity(ctx, orc, C, shape, P, G, seed):
    """The whole pipeline (Alg. 1/2) on a noisy phantom: same PSO trajectory
    (bit-identical lambda*, xi*), labels identical on >= 99.9% of voxels
    (north_star), centres within 1e-3.  Only asserted where the final IFCM is
    well conditioned (lambda*, xi* not both ~1)."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    vol, lab = _small_case(C=C, shape=shape, seed=11)
    cfg = IfcmConfig(C=C, eps=1e-5, max_iter=100)
    pso = PsoConfig(P=P, max_gen=G, patience=0, seed=seed)
    vt = torch.as_tensor(vol, device="cuda:0")
    labels, U, rep = ctx.segment(vt, cfg, pso, want_U=True)
    r = orc.segment_u8(vol, C=C, P=P, max_gen=G, seed=seed)
    assert np.abs(np.array(rep["c_init"]) - r.c_init).max() < 1e-6
    assert rep["lambda"] == r.lam and rep["xi"] == r.xi
    assert rep["generations"] == G
    if min(r.lam, r.xi) > 0.95:
        # ill-conditioned final IFCM: same-state parity from the GPU's final
        # state instead of comparing two chaotic trajectories (tests/illcond.py)
        from tests.illcond import final_state_step_parity
        final_state_step_parity(ctx, orc, torch.as_tensor(vol, device="cuda:0"), U, rep["centers"],
                                rep["lambda"], rep["xi"], cfg)
        return
    agree = (labels.cpu().numpy() == r.labels).mean()
    assert agree >= 0.999, agree
    assert np.allclose(rep["centers"], r.c, rtol=1e-3)
    assert abs(rep["final_iters"] - r.final_iters) <= 2


def test_segment_host_equals_device(ctx):
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    vol, _ = _small_case(C=3, shape=(8, 20, 20), seed=2)
    cfg = IfcmConfig(C=3)
    pso = PsoConfig(P=3, max_gen=3, patience=0, seed=5)
    vt = torch.as_tensor(vol, device="cuda:0")
    ws = ctx.workspace(20, 20, 8, cfg, pso)
    lab_d, _, rep_d = ctx.segment(vt, cfg, pso, ws=ws)
    vh = torch.as_tensor(vol).pin_memory()
    lh = torch.empty(vol.shape, dtype=torch.uint8).pin_memory()
    rep_h = ctx.segment_host(vh, cfg, pso, ws, lh)
    assert (lh.numpy() == lab_d.cpu().numpy()).all()
    assert rep_h["lambda"] == rep_d["lambda"]
    # z_slice: only that plane is written
    lab_z, _, _ = ctx.segment(vt, cfg, pso, ws=ws, z_slice=3)
    assert (lab_z.cpu().numpy() == lab_d.cpu().numpy()[3]).all()


def test_segment_determinism(ctx):
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    vol, _ = _small_case(C=4, shape=(12, 30, 33), seed=8)
    cfg = IfcmConfig(C=4)
    pso = PsoConfig(P=5, max_gen=4, patience=0, seed=3)
    vt = torch.as_tensor(vol, device="cuda:0")
    a = ctx.segment(vt, cfg, pso, want_U=True)
    b = ctx.segment(vt, cfg, pso, want_U=True)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    assert a[2]["J"] == b[2]["J"]


@pytest.mark.parametrize("eb", [1, 3, 5])
def test_eval_batch_bit_identical(ctx, eb):
    """pifcm_pso_cfg.eval_batch: CHAINED evaluation in launches of eb states
    over a pool of P + eb + 1 slots gives the same pipeline, bit for bit, as
    one launch over 2P + 1 slots."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    vol, _ = _small_case(C=4, shape=(9, 26, 30), seed=8)
    vt = torch.as_tensor(vol, device="cuda:0")
    cfg = IfcmConfig(C=4)
    base = PsoConfig(P=7, max_gen=4, patience=0, seed=3)
    bat = PsoConfig(P=7, max_gen=4, patience=0, seed=3, eval_batch=eb)
    nz, ny, nx = vol.shape
    slot = nz * ny * nx * 16
    assert ctx.workspace_size(nx, ny, nz, cfg, base) - ctx.workspace_size(nx, ny, nz, cfg, bat) >= (7 - eb) * slot
    la, Ua, ra = ctx.segment(vt, cfg, base, want_U=True)
    lb, Ub, rb = ctx.segment(vt, cfg, bat, want_U=True)
    assert torch.equal(la, lb) and torch.equal(Ua, Ub)
    for k in ("lambda", "xi", "J", "generations", "gbest_particle", "fcm_iters", "final_iters", "centers"):
        assert ra[k] == rb[k], k


def test_eval_batch_slab_bit_identical(ctx):
    """The same for the z-slab swarm (SlabSegmenter, one rank)."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import SlabSegmenter
    vol, _ = _small_case(C=4, shape=(21, 24, 27), seed=9)
    vt = torch.as_tensor(vol, device="cuda:0")
    out = []
    for eb in (0, 2):
        seg = SlabSegmenter(ctx, IfcmConfig(C=4), PsoConfig(P=5, max_gen=3, patience=0, seed=17, eval_batch=eb),
                            vol.shape)
        seg.keep_trace = True
        rep = seg.segment(vt)
        out.append((seg.labels.cpu().numpy(), rep, np.stack([t.numpy() for t in seg.trace])))
    (la, ra, ta), (lb, rb, tb) = out
    assert (la == lb).all() and (ta == tb).all()
    for k in ("lambda", "xi", "J", "generations", "gbest_particle", "final_iters", "centers"):
        assert ra[k] == rb[k], k
