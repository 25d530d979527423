"""Multi-process particle sharding on CPU (gloo, world_size 2): the sharded PSO
loop of paper_2002_01981_b200.dist, driven by an oracle-backed engine, must
reproduce the single-process oracle PSO exactly (same fitness vector every
generation, same gbest trajectory and result)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2002_01981_b200.dist import PsoOutcome, ShardedPso, allgather_fitness, shard_range


def test_shard_range():
    assert [shard_range(20, 8, r) for r in range(8)] == [
        (0, 3), (3, 6), (6, 9), (9, 12), (12, 14), (14, 16), (16, 18), (18, 20)]
    assert [shard_range(32, 1, 0)] == [(0, 32)]
    for P in range(1, 40):
        for w in range(1, 9):
            if w > P:
                continue
            rs = [shard_range(P, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == P
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


class OracleEngine:
    """ShardedPso engine whose fitness evaluations run the fp64 oracle step on
    this rank's particles (test double of GpuPsoEngine)."""

    def __init__(self, orc, x, U0, c0, P, seed):
        self.orc, self.x, self.U0, self.c0, self.P, self.seed = orc, x, U0, c0, P, seed

    def init(self, p0, p1):
        self.p0, self.p1 = p0, p1
        self.pos, self.vel = self.orc.pso_init(self.P, self.seed)
        self.pbf = np.full(self.P, np.inf)
        self.pbx = self.pos.copy()
        self.gbest = -1
        self.gen = 0
        self.U = {p: self.U0.copy() for p in range(p0, p1)}
        self.c = {p: self.c0.copy() for p in range(p0, p1)}
        self.local = np.zeros(p1 - p0)
        self.snap = None
        self.log = []

    def eval(self):
        for p in range(self.p0, self.p1):
            Un, cn, J, _ = self.orc.ifcm_step(self.x, self.U[p], self.c[p], self.pos[p, 0], self.pos[p, 1])
            self.U[p], self.c[p] = Un, cn
            self.local[p - self.p0] = J

    def local_fitness(self):
        return torch.tensor(self.local, dtype=torch.float64)

    def set_fitness(self, full):
        self.f = full.numpy().copy()
        self.log.append(self.f.copy())

    def update(self):
        eval_pos = self.pos.copy()
        self.gbest, imp = self.orc.pso_update(self.f, self.pos, self.vel, self.pbf, self.pbx, self.gbest,
                                              self.gen, self.seed)
        if imp:
            self.snap = (eval_pos[self.gbest, 0], eval_pos[self.gbest, 1], self.pbf[self.gbest])
        self.gen += 1

    def summary(self):
        lam, xi, J = self.snap
        return PsoOutcome(lam, xi, J, self.gen, self.gbest), False


def _problem(orc):
    from inputs import add_noise_u8, cube_phantom
    img, _ = cube_phantom(10, 9, 4, (0.1, 0.5, 0.9))
    x = add_noise_u8(img, 7.0, 3).astype(np.float64) / 255.0
    U0, c0, _ = orc.fcm_run(x, np.array([0.1, 0.5, 0.9]))
    return x, U0, c0


def _worker(rank, world, port, P, G, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    x, U0, c0 = _problem(oracle)
    eng = OracleEngine(oracle, x, U0, c0, P, seed)
    runner = ShardedPso(eng, P, dist)
    out = runner.run(G, early_stop=False)
    # gbest state lives on its owner
    owner = runner.owner_of(out.gbest_particle)
    has = int(out.gbest_particle in eng.U)
    # uneven all-gather sanity
    loc = torch.arange(runner.p0, runner.p1, dtype=torch.float64)
    full = allgather_fitness(dist, loc, P, world)
    q.put((rank, out.lam, out.xi, out.J, out.gbest_particle, out.generations, owner, has,
           np.array(eng.log), full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("P,world", [(5, 2), (6, 2)])
def test_sharded_pso_equals_single_process(orc, P, world):
    G, seed = 4, 2024
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, G, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, U0, c0 = _problem(orc)
    r = orc.pso_run(x, U0, c0, P=P, max_gen=G, seed=seed)
    for (rank, lam, xi, J, gb, gens, owner, has, log, full) in res:
        assert (lam, xi) == (r.lam, r.xi)
        assert J == r.J
        assert gens == G
        assert (log == r.trace_f).all()       # identical fitness vectors every generation
        assert (full == np.arange(P)).all()   # uneven ranges gathered in particle order
        assert has == (rank == owner)


def test_slab_range():
    from paper_2002_01981_b200.dist import slab_range
    assert [slab_range(181, 4, r, 16) for r in range(4)] == [(0, 48), (48, 48), (96, 48), (144, 37)]
    for nz in (1, 15, 16, 17, 40, 181, 512):
        for tz in (8, 16, 19):
            chunks = -(-nz // tz)
            for w in range(1, min(chunks, 8) + 1):
                rs = [slab_range(nz, w, r, tz) for r in range(w)]
                assert rs[0][0] == 0 and sum(n for _, n in rs) == nz
                assert all(z0 % tz == 0 and n > 0 for z0, n in rs)            # whole global chunks
                assert all(rs[i][0] + rs[i][1] == rs[i + 1][0] for i in range(w - 1))
                ch = [-(-n // tz) for _, n in rs]
                assert max(ch) - min(ch) <= 1


def test_slab_chunk_depends_on_the_volume_only():
    """pifcm_slab_chunk (host-only ABI query): >= 8 chunks where the volume
    allows (8 slabs get work), >= 8 planes per chunk, deterministic."""
    from paper_2002_01981_b200.api import PifcmError, slab_chunk
    for nx, ny, nz in [(181, 217, 181), (512, 512, 512), (37, 40, 50), (854, 854, 1), (30, 26, 12), (8, 8, 7)]:
        tz = slab_chunk(nx, ny, nz)
        chunks = -(-nz // tz)
        assert 1 <= tz <= nz
        assert chunks >= min(8, -(-nz // 8))
        assert tz >= 8 or chunks == 1 or tz * (chunks - 1) < nz
        assert slab_chunk(nx, ny, nz) == tz
    with pytest.raises(PifcmError):
        slab_chunk(0, 5, 5)


class _HostCtx:
    """The host-only part of a Context (pifcm_slab_chunk / pifcm_slab_records
    need no GPU) with CPU tensors, for the slab bookkeeping on CPU ranks."""
    torch_device = __import__("torch").device("cpu")

    def __init__(self):
        from paper_2002_01981_b200 import _abi
        self.lib = _abi.load()

    def slab_chunk(self, nx, ny, nz_total):
        from paper_2002_01981_b200.api import slab_chunk
        return slab_chunk(nx, ny, nz_total, self.lib)

    def slab_records(self, grid):
        import ctypes as ct
        n = ct.c_int32()
        assert self.lib.pifcm_slab_records(ct.byref(grid), ct.byref(n)) == 0
        return n.value


def _halo_worker(rank, world, port, H, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_01981_b200.dist import _SlabGeometry
    nx, ny, nz_total, P = 5, 4, 40, 2
    g = _SlabGeometry(_HostCtx(), nx, ny, nz_total, P, dist, H)
    pl = nx * ny
    # a state whose every voxel holds (state, global plane, voxel) in its row
    U = torch.full((P, (g.nz + 2 * H) * pl, 4), -1.0)
    for p in range(P):
        for k in range(g.nz):
            U[p, (H + k) * pl:(H + k + 1) * pl, 0] = p
            U[p, (H + k) * pl:(H + k + 1) * pl, 1] = g.z0 + k

    def pack(op, buf):  # the first / last H local planes (pifcm_slab_halo_v ops 0, 1)
        src = H if op == 0 else g.nz
        buf.copy_(U[:, src * pl:(src + H) * pl])

    def unpack(op, buf):  # the lower / upper H halo planes (ops 2, 3), zeros outside the volume
        dst = 0 if op == 2 else g.nz + H
        U[:, dst * pl:(dst + H) * pl] = 0.0 if buf is None else buf

    g.exchange(pack, unpack)
    q.put((rank, g.z0, g.nz, U.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [1, 2, 3])
def test_slab_halo_exchange_two_ranks(H):
    """The z-slab halo bookkeeping of the drivers (_SlabGeometry.exchange over
    gloo, world 2, CPU): every rank's H lower / upper halo planes hold the
    neighbour's global planes z0 - H .. z0 - 1 and z0 + nz .. z0 + nz + H - 1,
    zeros outside the volume (v = H shells, Eq. 9-10)."""
    import torch.multiprocessing as mp
    port = _free_port()
    cm = mp.get_context("spawn")
    q = cm.Queue()
    procs = [cm.Process(target=_halo_worker, args=(r, 2, port, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pl = 5 * 4
    for rank, z0, nz, U in res:
        for k in range(H):  # lower halo plane k = global plane z0 - H + k
            gz = z0 - H + k
            plane = U[:, k * pl:(k + 1) * pl]
            if gz < 0:
                assert (plane == 0).all()
            else:
                assert (plane[:, :, 1] == gz).all() and (plane[0, :, 0] == 0).all() and (plane[1, :, 0] == 1).all()
        for k in range(H):  # upper halo plane k = global plane z0 + nz + k
            gz = z0 + nz + k
            plane = U[:, (H + nz + k) * pl:(H + nz + k + 1) * pl]
            if gz >= 40:
                assert (plane == 0).all()
            else:
                assert (plane[:, :, 1] == gz).all()
