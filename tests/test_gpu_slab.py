"""z-slab sharding of the IFCM iteration: a volume split into
slabs with v halo planes per side (v = 1, 2) gives memberships bit-identical to the
whole-volume step and centres / J bit-identical for any number of slabs (the
reductions use global z-chunks fixed by the volume, pifcm_slab_chunk); across processes (gloo, two
ranks on one GPU) through the SlabIfcm driver."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from inputs import random_state

pytestmark = pytest.mark.gpu

NX, NY, NZ, C, P = 37, 40, 50, 4, 2


class _OneRank:
    def __init__(self, world, rank):
        self.w, self.r = world, rank

    def get_world_size(self):
        return self.w

    def get_rank(self):
        return self.r


def _state():
    x, U0, c0 = random_state(NX, NY, NZ, C, seed=21, crisp_frac=0.1)
    _, U1, c1 = random_state(NX, NY, NZ, C, seed=22)
    return x, np.stack([U0, U1]), np.stack([c0, c1])


def _virtual_slabs(ctx, world, iters, lx, v=1):
    """All slabs in one process: halos (v planes per side) copied between slab
    objects directly."""
    from paper_2002_01981_b200 import IfcmConfig, to_aos, to_pitched_x
    from paper_2002_01981_b200.dist import SlabIfcm
    x, U, c = _state()
    dev = torch.device("cuda:0")
    xt = to_pitched_x(x, dev)
    Ut = to_aos(U, dev)
    ct = torch.zeros((P, 4), device=dev)
    ct[:, :C] = torch.as_tensor(c)
    cfg = IfcmConfig(C=C, v=v)
    H = v
    slabs = []
    for r in range(world):
        s = SlabIfcm(ctx, cfg, NX, NY, NZ, P, dist=_OneRank(world, r))
        s.load_x(xt)
        s.load_state(Ut, ct)
        slabs.append(s)
    lxt = torch.tensor(lx, dtype=torch.float64, device=dev)
    pl = NX * NY
    for _ in range(iters):
        for i, s in enumerate(slabs):
            if i > 0:  # the lower neighbour's last H local planes
                nb = slabs[i - 1]
                s.geo.halo["recv_lo"].copy_(nb.Ua[:, nb.nz * pl:(nb.nz + H) * pl])
            if i < world - 1:  # the upper neighbour's first H local planes
                nb = slabs[i + 1]
                s.geo.halo["recv_hi"].copy_(nb.Ua[:, H * pl:2 * H * pl])
        for s in slabs:
            h = s.geo.halo
            s.ctx.slab_halo(s.grid, P, 2, s.Ua, h["recv_lo"] if s.rank > 0 else None, v=H)
            s.ctx.slab_halo(s.grid, P, 3, s.Ua, h["recv_hi"] if s.rank < world - 1 else None, v=H)
            s.ctx.slab_step(s.grid, cfg, s.x, s.Ua, s.Ub, s.centers, lxt, s.geo.rec)
            s.geo.rec_pad.zero_()
            s.geo.rec_pad[:, : s.geo.nrec] = s.geo.rec
        gathered = torch.stack([s.geo.rec_pad for s in slabs])
        for s in slabs:
            s.ctx.slab_finalize(C, P, world, s.geo.nrec_max, gathered, s.centers, stats=s.stats,
                                counts=s.geo.counts)
            s.Ua, s.Ub = s.Ub, s.Ua
    U_full = torch.cat([s.local_U() for s in slabs], dim=1)
    return U_full, slabs[0].centers.clone(), slabs[0].stats.clone(), [s.centers for s in slabs]


@pytest.mark.parametrize("v", [1, 2])
def test_slab_equals_whole_volume_and_is_g_invariant(v):
    """v = 2: two Chebyshev shells (Eq. 9-10), two halo planes per side."""
    from paper_2002_01981_b200 import Context, IfcmConfig, to_aos, to_pitched_x
    ctx = Context(0)
    lx = [[0.6, 0.8], [1.0, 1.0]]
    U1, c1, st1, _ = _virtual_slabs(ctx, 1, 3, lx, v=v)
    U3, c3, st3, cs = _virtual_slabs(ctx, 3, 3, lx, v=v)
    assert (U1 == U3).all()                       # memberships: per voxel, identical
    assert (c1 == c3).all() and (st1 == st3).all()  # reductions: G-invariant
    for c in cs:
        assert (c == c3).all()                    # every rank holds the same centres
    # against the whole-volume step: memberships bit-identical, centres ~1e-7 (other grouping)
    x, U, c = _state()
    dev = torch.device("cuda:0")
    Uin = to_aos(U, dev)
    Uo = torch.empty_like(Uin)
    cen = torch.zeros((P, 4), device=dev)
    cen[:, :C] = torch.as_tensor(c)
    lxt = torch.tensor(lx, dtype=torch.float64, device=dev)
    ctx.iterate(to_pitched_x(x, dev), Uin, Uo, cen, lxt, IfcmConfig(C=C, v=v), iters=3, nx=NX)
    assert torch.equal(Uo, U3)
    assert torch.allclose(cen, c3, rtol=1e-6, atol=0)


@pytest.mark.parametrize("v", [1, 2])
def test_slab_parity_with_oracle(orc, v):
    """One slab step from the same state vs the fp64 oracle (1e-4 / 1e-4)."""
    x, U, c = _state()
    U3, c3, st3, _ = _virtual_slabs(__import__("paper_2002_01981_b200").Context(0), 3, 1, [[0.4, 0.7], [0.9, 0.2]],
                                    v=v)
    for p, (l, s) in enumerate([(0.4, 0.7), (0.9, 0.2)]):
        Uo, co, Jo, _ = orc.ifcm_step(x, U[p], c[p], l, s, v=v, h=1.0)
        assert np.abs(U3[p, :, :C].cpu().numpy() - Uo).max() < 1e-4
        assert np.all(np.abs(c3[p, :C].cpu().numpy() - co) <= 1e-4 * np.abs(co))
        assert abs(st3[p, 0].item() - Jo) <= 1e-4 * Jo


def _worker(rank, world, port, q, v=1):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_01981_b200 import Context, IfcmConfig, to_aos, to_pitched_x
    from paper_2002_01981_b200.dist import SlabIfcm
    ctx = Context(0)
    x, U, c = _state()
    dev = torch.device("cuda:0")
    s = SlabIfcm(ctx, IfcmConfig(C=C, v=v), NX, NY, NZ, P, dist)
    s.load_x(to_pitched_x(x, dev))
    ct = torch.zeros((P, 4), device=dev)
    ct[:, :C] = torch.as_tensor(c)
    s.load_state(to_aos(U, dev), ct)
    s.run(torch.tensor([[0.6, 0.8], [1.0, 1.0]], dtype=torch.float64, device=dev), iters=3)
    q.put((rank, s.z0, s.local_U().cpu().numpy(), s.centers.cpu().numpy(), s.stats.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("v", [1, 2])
def test_slab_driver_two_ranks(v):
    from paper_2002_01981_b200 import Context
    ctx = Context(0)
    U1, c1, st1, _ = _virtual_slabs(ctx, 1, 3, [[0.6, 0.8], [1.0, 1.0]], v=v)
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cm = mp.get_context("spawn")
    q = cm.Queue()
    procs = [cm.Process(target=_worker, args=(r, 2, port, q, v)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    U = np.concatenate([r[2] for r in res], axis=1)
    assert (U == U1.cpu().numpy()).all()
    for r in res:
        assert (r[3] == c1.cpu().numpy()).all() and (r[4] == st1.cpu().numpy()).all()
