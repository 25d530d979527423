"""GPU parity of the ANCHORED and LEADER fitness modes (
reading R22) against the fp64 oracle: the particle-invariant H, F pass plus
the pointwise swarm evaluation, the snapshot / advance steps in the update,
and the whole pipeline with each mode; sharded over two ranks (gloo) equal to
one process."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ANCHORED, LEADER = 1, 2


@pytest.fixture(scope="module")
def ctx():
    from paper_2002_01981_b200 import Context
    return Context(0)


def _case(C=3, shape=(10, 24, 28), seed=4):
    from inputs import add_noise_u8, cube_phantom
    nz, ny, nx = shape
    img, lab = cube_phantom(nx, ny, nz, (0.1, 0.5, 0.9) if C == 3 else (0.1, 0.35, 0.65, 0.9))
    return add_noise_u8(img, 7.0, seed), lab


def _swarm(ctx, orc, P, seed, mode, C=3, shape=(10, 24, 28), v=1):
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig, to_aos, to_pitched_x
    from paper_2002_01981_b200.api import _grid
    vol, _ = _case(C, shape)
    x = vol.astype(np.float32) / 255.0
    Uf, cf, _ = orc.fcm_run(x, np.linspace(0.1, 0.9, C))
    U0, c0 = Uf.astype(np.float32), cf.astype(np.float32)
    nz, ny, nx = x.shape
    dev = torch.device("cuda:0")
    cfg = IfcmConfig(C=C, v=v)
    pso = PsoConfig(P=P, max_gen=50, patience=0, seed=seed, fitness=mode)
    xt, Ut = to_pitched_x(x, dev), to_aos(U0, dev)
    c4 = torch.zeros(4, device=dev)
    c4[:C] = torch.as_tensor(c0)
    ws = ctx.workspace(nx, ny, nz, cfg, pso)
    g = _grid(nx, ny, nz)
    ctx.pso_init(g, cfg, pso, Ut, c4, ws)
    return x, U0, c0, cfg, pso, xt, Ut, ws, g


@pytest.mark.parametrize("mode,G,P,seed,v", [(ANCHORED, 6, 6, 777, 1), (ANCHORED, 4, 40, 5, 1), (LEADER, 3, 6, 91, 1),
                                             (LEADER, 3, 33, 12, 1), (ANCHORED, 4, 6, 777, 2), (LEADER, 3, 6, 91, 2)])
def test_mode_eval_parity(ctx, orc, mode, G, P, seed, v):
    """Every generation's fitness vector within 1e-5 of the oracle's (ANCHORED
    evaluates every generation from the same start; LEADER's shared state
    drifts by fp32 rounding: 1e-5 for generation 0, 1e-4 after), identical
    gbest sequence and (lambda*, xi*), and the gbest snapshot of Alg. 1 step
    10 within 1e-4."""
    x, U0, c0, cfg, pso, xt, Ut, ws, g = _swarm(ctx, orc, P, seed, mode, v=v)
    fit = ctx.pso_fitness(g, cfg, pso, ws)
    r = orc.pso_run(x, U0, c0, P=P, max_gen=G, seed=seed, fitness_mode=mode, v=v)
    for gen in range(G):
        ctx.pso_eval(g, cfg, pso, xt, ws)
        f = fit.cpu().numpy()
        tol = 1e-5 if (mode == ANCHORED or gen == 0) else 1e-4
        assert np.allclose(f, r.trace_f[gen], rtol=tol, atol=0), (gen, np.abs(f / r.trace_f[gen] - 1).max())
        ctx.pso_update(g, cfg, pso, ws, x=xt)
        summ, _ = ctx.pso_result(g, cfg, pso, ws)
        assert summ.gbest_particle == r.trace_gbest[gen]
    assert summ.lam == r.lam and summ.xi == r.xi
    assert abs(summ.J - r.J) <= 1e-4 * r.J
    Ug = torch.empty_like(Ut)
    cg = torch.empty(4, device=Ut.device)
    ctx.pso_gbest_state(g, cfg, pso, ws, Ug, cg)
    assert np.abs(Ug.cpu().numpy()[:, :3] - r.U).max() < 1e-4
    assert np.allclose(cg.cpu().numpy()[:3], r.c, rtol=1e-4)


@pytest.mark.parametrize("mode,G,seed,v", [(ANCHORED, 4, 3, 1), (LEADER, 4, 3, 1), (ANCHORED, 2, 1, 1), (LEADER, 2, 1, 1),
                                          (ANCHORED, 3, 3, 2), (LEADER, 3, 1, 2)])
def test_mode_segment_parity(ctx, orc, mode, G, seed, v):
    """The whole pipeline with the mode: same GMM start and PSO trajectory
    (bit-identical lambda*, xi*); labels >= 99.9 % where the final IFCM is well
    conditioned."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    vol, _ = _case(C=4, shape=(12, 30, 33), seed=8)
    cfg = IfcmConfig(C=4, v=v)
    pso = PsoConfig(P=6, max_gen=G, patience=0, seed=seed, fitness=mode)
    labels, U, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), cfg, pso, want_U=True)
    r = orc.segment_u8(vol, C=4, P=6, max_gen=G, seed=seed, fitness_mode=mode, v=v)
    assert rep["lambda"] == r.lam and rep["xi"] == r.xi
    if min(r.lam, r.xi) > 0.95:
        # ill-conditioned final IFCM: same-state parity from the GPU's final
        # state instead of comparing two chaotic trajectories (tests/illcond.py)
        from tests.illcond import final_state_step_parity
        final_state_step_parity(ctx, orc, torch.as_tensor(vol, device="cuda:0"), U, rep["centers"],
                                rep["lambda"], rep["xi"], cfg)
        return
    agree = (labels.cpu().numpy() == r.labels).mean()
    assert agree >= 0.999, agree
    # centres after up to 100 final-IFCM iterations from different roundings;
    # the 124-neighbour map (v = 2) drifts further than v = 1's (the per-step
    # parity from the same state is 1e-4: test_step_parity_v2)
    rtol = 1e-3 if v == 1 else 1e-2
    assert np.allclose(rep["centers"], r.c, rtol=rtol), (rep["centers"], r.c, r.lam, r.xi)


def test_mode_workspace_is_smaller(ctx):
    """ANCHORED / LEADER keep 2 / 3 state slots instead of CHAINED's 2P + 1."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    cfg = IfcmConfig(C=4)
    n = {m: ctx.workspace_size(181, 217, 181, cfg, PsoConfig(P=32, fitness=m)) for m in (0, ANCHORED, LEADER)}
    slot = 181 * 217 * 181 * 16
    assert n[0] > 60 * slot and n[ANCHORED] < 5 * slot and n[LEADER] < 6 * slot


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import ShardedSegmenter
    ctx = Context(0)
    vol, _ = _case(C=4, shape=(20, 26, 30), seed=6)
    seg = ShardedSegmenter(ctx, IfcmConfig(C=4), PsoConfig(P=5, max_gen=4, patience=0, seed=31, fitness=mode),
                           vol.shape, dist)
    rep = seg.segment(torch.as_tensor(vol, device="cuda:0"))
    q.put((rank, seg.labels.cpu().numpy(), rep["lambda"], rep["xi"], rep["centers"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [ANCHORED, LEADER])
def test_mode_sharded_equals_single(ctx, mode):
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    vol, _ = _case(C=4, shape=(20, 26, 30), seed=6)
    lab, _, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), IfcmConfig(C=4),
                              PsoConfig(P=5, max_gen=4, patience=0, seed=31, fitness=mode))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cm = mp.get_context("spawn")
    q = cm.Queue()
    procs = [cm.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, labels, lam, xi, cen in res:
        assert (lam, xi) == (rep["lambda"], rep["xi"])
        assert (labels == lab.cpu().numpy()).all()
        assert cen == rep["centers"]
