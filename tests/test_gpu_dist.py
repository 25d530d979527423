"""G-invariance of the particle-sharded pipeline on one GPU: two ranks (gloo,
both on cuda:0) running ShardedSegmenter must give labels bit-identical to
the single-process pifcm_segment; world_size 1 likewise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _case(nz):
    from inputs import add_noise_u8, cube_phantom
    img, _ = cube_phantom(30, 26, nz, (0.1, 0.35, 0.65, 0.9))
    return add_noise_u8(img, 7.0, 6)


CFG = dict(C=4)
PSO = dict(P=5, max_gen=4, patience=0, seed=31)


def _worker(rank, world, port, nz, shard, q, eb=0):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import ShardedSegmenter
    ctx = Context(0)
    vol = _case(nz)
    seg = ShardedSegmenter(ctx, IfcmConfig(**CFG), PsoConfig(**PSO, eval_batch=eb), vol.shape, dist,
                           shard_final=shard)
    rep = seg.segment(torch.as_tensor(vol, device="cuda:0"))
    q.put((rank, seg.labels.cpu().numpy(), rep["lambda"], rep["xi"], rep["final_iters"], rep["centers"]))
    dist.barrier()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# nz = 12: one z-chunk, the final IFCM runs replicated; nz = 40: five chunks,
# the final IFCM z-slab sharded 3 + 2 (uneven record counts) or replicated
# eb: each rank evaluates its particles in batches of eb over Pl + eb + 1 slots
@pytest.mark.parametrize("nz,shard,eb", [(12, None, 0), (40, True, 0), (40, False, 0), (40, True, 1)])
def test_sharded_equals_single(nz, shard, eb):
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    from paper_2002_01981_b200.dist import ShardedSegmenter
    ctx = Context(0)
    vol = _case(nz)
    vt = torch.as_tensor(vol, device="cuda:0")
    lab, _, rep = ctx.segment(vt, IfcmConfig(**CFG), PsoConfig(**PSO))
    ref = lab.cpu().numpy()
    # world_size 1 (no process group)
    seg = ShardedSegmenter(ctx, IfcmConfig(**CFG), PsoConfig(**PSO), vol.shape, None)
    r1 = seg.segment(vt)
    assert (seg.labels.cpu().numpy() == ref).all()
    assert (r1["lambda"], r1["xi"]) == (rep["lambda"], rep["xi"])
    assert r1["final_iters"] == rep["final_iters"] and r1["fcm_iters"] == rep["fcm_iters"]
    assert r1["centers"] == rep["centers"]
    # two ranks on the same GPU (gloo collectives through host memory)
    cm = mp.get_context("spawn")
    q = cm.Queue()
    port = _port()
    procs = [cm.Process(target=_worker, args=(r, 2, port, nz, shard, q, eb)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, labels, lam, xi, fi, cen in res:
        assert (labels == ref).all()
        assert (lam, xi) == (rep["lambda"], rep["xi"])
        assert fi == rep["final_iters"] and cen == rep["centers"]


def _abi_worker(rank, world, port, P, q):
    """pifcm_segment itself sharded through the C ABI's communicator (the
    library calls back into gloo for the fitness all-gather and the gbest
    broadcast; NCCL would be the same calls on separate GPUs)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dataclasses import replace
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    ctx = Context(0)
    ctx.attach_dist(rank, world, backend="host")
    vol = _case(40)
    pso = PsoConfig(**dict(PSO, P=P))
    a, b = ctx.dist_range(P, world, rank)
    pso = replace(pso, p_begin=a, p_end=b)
    lab, _, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), IfcmConfig(**CFG), pso)
    q.put((rank, lab.cpu().numpy(), rep["lambda"], rep["xi"], rep["final_iters"], rep["centers"],
           rep["gbest_particle"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P,world", [(5, 2), (7, 3)])
def test_abi_sharded_segment_equals_single(P, world):
    """SURVEY 8(b)'s pifcm_dist: every rank's pifcm_segment returns the
    single-process labels, (lambda*, xi*), final iterations and centres bit
    for bit, for uneven particle splits (5 over 2, 7 over 3)."""
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    ctx = Context(0)
    vol = _case(40)
    lab, _, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), IfcmConfig(**CFG),
                              PsoConfig(**dict(PSO, P=P)))
    ref = lab.cpu().numpy()
    cm = mp.get_context("spawn")
    q = cm.Queue()
    port = _port()
    procs = [cm.Process(target=_abi_worker, args=(r, world, port, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, labels, lam, xi, fi, cen, gb in res:
        assert (labels == ref).all(), rank
        assert (lam, xi) == (rep["lambda"], rep["xi"])
        assert fi == rep["final_iters"] and cen == rep["centers"] and gb == rep["gbest_particle"]
