"""PSO-3DPIFCM over z-slab ranks (the C5 workload): the slab
swarm's fitness against the fp64 oracle, the whole slab pipeline against the
oracle's pipeline, bit-identical results for one and two ranks (gloo, both
on cuda:0), and the C5 shape (512^3) end to end with properties that hold at
any size."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2002_01981_b200 import Context
    return Context(0)


def _case(C, shape, seed=4):
    from inputs import add_noise_u8, cube_phantom
    nz, ny, nx = shape
    img, lab = cube_phantom(nx, ny, nz, (0.1, 0.5, 0.9) if C == 3 else (0.1, 0.35, 0.65, 0.9))
    return add_noise_u8(img, 7.0, seed), lab


def test_slab_pso_eval_parity(ctx, orc):
    """Generations 0 and 1 of the slab swarm (CHAINED fitness, one step per
    particle from its own state) within 1e-5 / 1e-4 of the oracle's PSO run,
    same gbest sequence, and the gbest state of Alg. 1 step 10."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig, to_aos, to_pitched_x
    from paper_2002_01981_b200.dist import SlabPso
    C, P, seed = 3, 6, 777
    vol, _ = _case(C, (10, 24, 28))
    x = vol.astype(np.float32) / 255.0
    Uf, cf, _ = orc.fcm_run(x, np.linspace(0.1, 0.9, C))
    U0, c0 = Uf.astype(np.float32), cf.astype(np.float32)
    nz, ny, nx = x.shape
    dev = torch.device("cuda:0")
    cfg = IfcmConfig(C=C)
    pso = PsoConfig(P=P, max_gen=50, patience=0, seed=seed)
    sw = SlabPso(ctx, cfg, pso, nx, ny, nz)
    geo = sw.geo
    xs = geo.slab_planes(to_pitched_x(x, dev))
    Us = geo.slab_planes(to_aos(U0, dev).view(nz, ny * nx, 4)).view(-1, 4)
    c4 = torch.zeros(4, device=dev)
    c4[:C] = torch.as_tensor(c0)
    sw.init(Us, c4)
    r = orc.pso_run(x, U0, c0, P=P, max_gen=2, seed=seed)
    for gen, tol in ((0, 1e-5), (1, 1e-4)):
        sw.generation(xs)
        f = sw.fitness().cpu().numpy()
        assert np.allclose(f, r.trace_f[gen], rtol=tol, atol=0), (gen, f, r.trace_f[gen])
        summ, _ = ctx.slab_pso_result(sw.grid, cfg, sw.pso, sw.ws)
        assert summ.gbest_particle == r.trace_gbest[gen]
    assert summ.lam == r.lam and summ.xi == r.xi
    assert abs(summ.J - r.J) <= 1e-4 * r.J
    Ug = torch.empty_like(Us)
    cg = torch.empty(4, device=dev)
    sw.gbest_state(Ug, cg)
    Ul = Ug.view(nz + 2, ny * nx, 4)[1: nz + 1].reshape(-1, 4)
    assert np.abs(Ul.cpu().numpy()[:, :C] - r.U).max() < 1e-4


@pytest.mark.parametrize("C,shape,P,G,seed,v", [(3, (20, 24, 28), 4, 3, 99, 1), (4, (26, 33, 35), 5, 2, 1, 1),
                                                (4, (20, 26, 30), 4, 2, 7, 2)])
def test_slab_segmenter_oracle(ctx, orc, C, shape, P, G, seed, v):
    """The whole slab pipeline against the oracle's Alg. 1 / Alg. 2: same GMM
    start, same PSO trajectory (bit-identical lambda*, xi*), labels identical
    on >= 99.9 % of voxels and centres within 1e-3 where the final IFCM is
    well conditioned."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import SlabSegmenter
    vol, _ = _case(C, shape, seed=11)
    cfg = IfcmConfig(C=C, eps=1e-5, max_iter=100, v=v)
    pso = PsoConfig(P=P, max_gen=G, patience=0, seed=seed)
    seg = SlabSegmenter(ctx, cfg, pso, vol.shape)
    rep = seg.segment(torch.as_tensor(vol, device="cuda:0"))
    r = orc.segment_u8(vol, C=C, P=P, max_gen=G, seed=seed, v=v)
    assert np.abs(np.array(rep["c_init"]) - r.c_init).max() < 1e-6
    assert rep["lambda"] == r.lam and rep["xi"] == r.xi
    assert rep["generations"] == G
    if min(r.lam, r.xi) > 0.95:
        # ill-conditioned final IFCM: same-state parity instead (tests/illcond.py)
        from tests.illcond import final_state_step_parity
        final_state_step_parity(ctx, orc, torch.as_tensor(vol, device="cuda:0"), seg.ifcm.local_U()[0].reshape(-1, 4),
                                rep["centers"], rep["lambda"], rep["xi"], cfg)
        return
    agree = (seg.labels.cpu().numpy() == r.labels).mean()
    assert agree >= 0.999, agree
    # centres after up to 100 final-IFCM iterations from different roundings;
    # the 124-neighbour map (v = 2) drifts further (as test_mode_segment_parity)
    assert np.allclose(rep["centers"], r.c, rtol=1e-3 if v == 1 else 1e-2)


def _worker(rank, world, port, shape, q, v=1):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import SlabSegmenter
    ctx = Context(0)
    vol, _ = _case(4, shape, seed=6)
    seg = SlabSegmenter(ctx, IfcmConfig(C=4, v=v), PsoConfig(P=5, max_gen=4, patience=0, seed=31), vol.shape,
                        dist)
    seg.keep_trace = True
    rep = seg.segment(torch.as_tensor(vol, device="cuda:0"))
    q.put((rank, seg.labels.cpu().numpy(), rep, np.stack([t.numpy() for t in seg.trace]),
           seg.geo.z0, seg.geo.nz))
    dist.barrier()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("v", [1, 2])
def test_slab_segmenter_g_invariant(ctx, v):
    """One rank and two ranks (2 + 1 z-chunks, uneven) give bit-identical
    labels, lambda*, xi*, J, centres, iteration counts and fitness traces
    (v = 2: two halo planes per side exchanged every generation / iteration)."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import SlabSegmenter
    shape = (40, 26, 30)
    vol, _ = _case(4, shape, seed=6)
    seg = SlabSegmenter(ctx, IfcmConfig(C=4, v=v), PsoConfig(P=5, max_gen=4, patience=0, seed=31), vol.shape)
    seg.keep_trace = True
    ref = seg.segment(torch.as_tensor(vol, device="cuda:0"))
    ref_lab = seg.labels.cpu().numpy()
    ref_tr = np.stack([t.numpy() for t in seg.trace])
    cm = mp.get_context("spawn")
    q = cm.Queue()
    port = _port()
    procs = [cm.Process(target=_worker, args=(r, 2, port, shape, q, v)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][4] == 0 and res[1][4] == res[0][5] and res[0][5] + res[1][5] == shape[0]
    for rank, labels, rep, tr, _, _ in res:
        assert (labels == ref_lab).all()
        assert (tr == ref_tr).all()
        for k in ("lambda", "xi", "J", "generations", "gbest_particle", "fcm_iters", "final_iters", "c_init",
                  "centers"):
            assert rep[k] == ref[k], (k, rep[k], ref[k])


def test_c5_shape_end_to_end(ctx, orc):
    """The C5 volume (512^3, 4 nested cubes, 7 % noise) through the slab
    pipeline on one rank with a reduced swarm (P = 4, 2 generations; the
    configured P = 64 needs >= 2 GPUs): labels in range, rows of U sum to 1,
    the final centres are Eq. 3 of the final memberships (oracle, fp64), the
    GMM start equals the oracle's."""
    from inputs import config_volume
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import SlabSegmenter
    vol, _ = config_volume("C5")
    cfg = IfcmConfig(C=4, max_iter=100)
    pso = PsoConfig(P=4, max_gen=2, patience=0, seed=12345)
    seg = SlabSegmenter(ctx, cfg, pso, vol.shape)
    rep = seg.segment(torch.as_tensor(vol, device="cuda:0"))
    c0 = orc.gmm_init(orc.histogram_u8(vol), 4)
    assert np.abs(np.array(rep["c_init"]) - c0).max() < 1e-6
    lab = seg.labels.cpu().numpy()
    assert lab.shape == vol.shape and lab.max() <= 3
    U = seg.ifcm.local_U()[0].cpu().numpy()
    assert np.abs(U.sum(1) - 1).max() < 1e-5
    x = orc.normalize_u8(vol).astype(np.float32)
    cE = orc.centers(x, U.astype(np.float64), np.zeros(4))
    assert np.all(np.abs(np.array(rep["centers"]) - cE) <= 1e-4 * np.abs(cE))
    assert (lab.ravel()[:: 997] == orc.argmax(U[:: 997].astype(np.float64))).all()
    assert 0 <= rep["lambda"] <= 1 and 0 <= rep["xi"] <= 1
