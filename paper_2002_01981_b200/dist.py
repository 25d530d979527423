"""Particle-sharded PSO-3DPIFCM across ranks (one process per GPU).

The PSO of Alg. 1 steps 3-9 evaluates every particle
independently (the fitness of particle p is one IFCM step of its own state at
its own (lambda, xi), CHAINED reading R11), so the particles are sharded over
ranks: rank r owns particles [p0, p1) and their membership states.  The only
exchanges are
  * an all-gather of the per-particle fitness (P doubles) every generation,
    after which every rank runs the same deterministic PSO update (so no
    positions are exchanged), and
  * a broadcast of the gbest state (its U and centres, Alg. 1 step 10) from
    the rank that owns the gbest particle, before the final IFCM (step 11).
The collectives go through torch.distributed (NCCL on GPUs); every compute
step runs in libpifcm.so.  The PSO loop is written against a small engine
interface so the sharding logic can be exercised on CPU (gloo) in tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["shard_range", "allgather_fitness", "ShardedPso", "GpuPsoEngine", "ShardedSegmenter",
           "slab_range", "SlabIfcm", "SlabIfcmP2P", "SlabPso", "SlabSegmenter"]


def shard_range(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, as-even-as-possible split of P particles over `world` ranks
    (20 over 8 -> 3,3,3,3,2,2,2,2)."""
    base, rem = divmod(P, world)
    p0 = rank * base + min(rank, rem)
    return p0, p0 + base + (1 if rank < rem else 0)


def allgather_fitness(dist, local: torch.Tensor, P: int, world: int) -> torch.Tensor:
    """All-gather the fp64 fitness of every rank's particle range into [P]
    (rank order = particle order).  Uneven ranges are padded to the largest."""
    if world == 1:
        return local.clone()
    maxl = -(-P // world)
    dev = local.device
    cpu_coll = dist.get_backend() == "gloo" and dev.type == "cuda"
    buf = torch.zeros(maxl, dtype=torch.float64, device="cpu" if cpu_coll else dev)
    buf[: local.numel()] = local.to(buf.device)
    out = torch.empty(world * maxl, dtype=torch.float64, device=buf.device)
    dist.all_gather_into_tensor(out, buf)
    parts = []
    for r in range(world):
        a, b = shard_range(P, world, r)
        parts.append(out[r * maxl: r * maxl + (b - a)])
    return torch.cat(parts).to(dev)


def broadcast_(dist, t: torch.Tensor, src: int):
    """Broadcast in place (through host memory when gloo carries CUDA tensors)."""
    if dist.get_backend() == "gloo" and t.device.type == "cuda":
        h = t.cpu()
        dist.broadcast(h, src=src)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src)


@dataclass
class PsoOutcome:
    lam: float
    xi: float
    J: float
    generations: int
    gbest_particle: int


class ShardedPso:
    """Generation loop of Alg. 1 steps 4-9 over sharded particles.

    engine must provide: init(p0, p1); eval(); local_fitness() -> Tensor[p1-p0];
    set_fitness(Tensor[P]); update(); summary() -> (PsoOutcome, stopped)."""

    def __init__(self, engine, P: int, dist=None, check_every: int = 4):
        self.engine = engine
        self.P = P
        self.dist = dist
        self.world = dist.get_world_size() if dist is not None else 1
        self.rank = dist.get_rank() if dist is not None else 0
        self.p0, self.p1 = shard_range(P, self.world, self.rank)
        self.check_every = check_every

    def run(self, max_gen: int, early_stop: bool) -> PsoOutcome:
        e = self.engine
        e.init(self.p0, self.p1)
        for gen in range(max_gen):
            e.eval()
            full = allgather_fitness(self.dist, e.local_fitness(), self.P, self.world)
            e.set_fitness(full)
            e.update()
            if early_stop and (gen + 1) % self.check_every == 0:
                _, stopped = e.summary()
                if stopped:
                    break
        out, _ = e.summary()
        return out

    def owner_of(self, particle: int) -> int:
        for r in range(self.world):
            a, b = shard_range(self.P, self.world, r)
            if a <= particle < b:
                return r
        raise ValueError(particle)


class GpuPsoEngine:
    """ShardedPso engine over libpifcm.so (pifcm_pso_init/eval/update)."""

    def __init__(self, ctx, grid, cfg, pso, x, U0, c0):
        self.ctx, self.grid, self.cfg, self.pso0 = ctx, grid, cfg, pso
        self.x, self.U0, self.c0 = x, U0, c0
        self.ws = None

    def init(self, p0, p1):
        from dataclasses import replace
        self.pso = replace(self.pso0, p_begin=p0, p_end=p1)
        if p0 == 0 and p1 == self.pso.P:
            self.pso = replace(self.pso, p_begin=0, p_end=0)
        self.p0, self.p1 = p0, p1
        g = self.grid
        n = self.ctx.workspace_size(g.nx, g.ny, g.nz, self.cfg, self.pso)
        if self.ws is None or self.ws.numel() < n:
            self.ws = torch.empty(n, dtype=torch.uint8, device=self.x.device)
        self.ctx.pso_init(g, self.cfg, self.pso, self.U0, self.c0, self.ws)
        self.fit = self.ctx.pso_fitness(g, self.cfg, self.pso, self.ws)

    def eval(self):
        self.ctx.pso_eval(self.grid, self.cfg, self.pso, self.x, self.ws)

    def local_fitness(self):
        return self.fit[self.p0:self.p1]

    def set_fitness(self, full):
        self.fit.copy_(full)

    def update(self):
        self.ctx.pso_update(self.grid, self.cfg, self.pso, self.ws, x=self.x)

    def summary(self):
        s, stopped = self.ctx.pso_result(self.grid, self.cfg, self.pso, self.ws)
        return PsoOutcome(s.lam, s.xi, s.J, s.generations, s.gbest_particle), stopped

    def gbest_state(self, U_out, c_out):
        self.ctx.pso_gbest_state(self.grid, self.cfg, self.pso, self.ws, U_out, c_out)


def _slab_driver(ctx, cfg, nx, ny, nz_total, P, dist):
    """SlabIfcmP2P (exchange over peer memory) where every rank can map the
    others' memory (decided collectively), else SlabIfcm (host-driven
    collectives); the results are the same."""
    try:
        return SlabIfcmP2P(ctx, cfg, nx, ny, nz_total, P, dist)
    except RuntimeError:
        return SlabIfcm(ctx, cfg, nx, ny, nz_total, P, dist)


class ShardedSegmenter:
    SHARD_FINAL_MIN_VOXELS = 4 * 1024 * 1024

    """pifcm_segment with the PSO particles sharded over the ranks of `dist`.

    Every rank normalises, fits the GMM and runs the FCM start (identical,
    deterministic), the PSO generations are sharded, the gbest state is
    broadcast from its owner, and the final IFCM runs either z-slab sharded
    (SlabIfcm, each rank's slab labels all-gathered; large volumes) or whole on
    every rank.  Both use the canonical z-chunk decomposition of
    pifcm_segment's final IFCM, so labels are bit-identical to the
    single-process pifcm_segment for any world size."""

    def __init__(self, ctx, cfg, pso, shape, dist=None, shard_final=None):
        """shard_final: None = by size (SHARD_FINAL_MIN_VOXELS), True / False force."""
        self.ctx, self.cfg, self.pso = ctx, cfg, pso
        self.nz, self.ny, self.nx = shape
        self.dist = dist
        self.dev = torch.device(f"cuda:{ctx.device}")
        nvox = self.nx * self.ny * self.nz
        self.Ub = torch.empty((1, nvox, 4), dtype=torch.float32, device=self.dev)
        self.Ua = torch.zeros((1, nvox, 4), dtype=torch.float32, device=self.dev)
        self.cen = torch.empty((1, 4), dtype=torch.float32, device=self.dev)
        self.mm = torch.zeros(64, dtype=torch.int32, device=self.dev)  # normalise's raw {min, max}
        self.engine = None
        world = dist.get_world_size() if dist is not None else 1
        tz = ctx.slab_chunk(self.nx, self.ny, self.nz)
        # The final IFCM (one state) runs z-slab sharded (exchange over peer
        # memory, a few tens of us per iteration) when a rank's share of an
        # iteration outweighs that; otherwise every rank runs it whole, in
        # the same canonical decomposition -- the results are bit-identical
        # either way.
        big = nvox >= self.SHARD_FINAL_MIN_VOXELS if shard_final is None else bool(shard_final)
        self.shard_final = world > 1 and -(-self.nz // tz) >= world and big
        self.slab = (_slab_driver(ctx, cfg, self.nx, self.ny, self.nz, 1, dist) if self.shard_final
                     else SlabIfcm(ctx, cfg, self.nx, self.ny, self.nz, 1, None))
        w = self.slab.world
        self.lab_counts = [slab_range(self.nz, w, r, tz)[1] * self.nx * self.ny for r in range(w)]
        self.lab_pad = torch.zeros((w, max(self.lab_counts)), dtype=torch.uint8, device=self.dev)

    def segment(self, vol: torch.Tensor) -> dict:
        from .api import _grid
        ctx, cfg = self.ctx, self.cfg
        nz, ny, nx = self.nz, self.ny, self.nx
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        # Alg. 2 step 1 + Alg. 1 step 2: normalise, GMM, FCM start (lambda = xi = 0)
        if vol.dtype not in (torch.uint8, torch.uint16):
            raise TypeError("the particle-sharded pipeline takes uint8 / uint16 volumes")
        x, hist = ctx.normalize(vol, mm=self.mm)
        c0 = ctx.gmm_init(hist, cfg.C)
        ev[1].record()
        # FCM start on the value histogram (R24), exactly as pifcm_segment
        counts = ctx.value_hist(vol)
        c_prev, c_fcm4, fst = ctx.fcm_hist(counts, self.mm, c0, cfg)
        ctx.fcm_memberships(x, c_prev, cfg.C, cfg.m, nx, U=self.Ub[0])
        self.cen.copy_(c_fcm4.view(1, 4))
        stats = torch.zeros((1, 4), dtype=torch.float64, device=self.dev)
        fcm_iters = int(fst[2].item())
        ev[2].record()
        # Alg. 1 steps 3-10: sharded PSO from (U_fcm, c_fcm)
        g = _grid(nx, ny, nz)
        U0 = self.Ub[0]
        c_fcm = self.cen[0].clone()
        self.engine = GpuPsoEngine(ctx, g, cfg, self.pso, x, U0, c_fcm)
        runner = ShardedPso(self.engine, self.pso.P, self.dist)
        out = runner.run(self.pso.max_gen, early_stop=self.pso.patience > 0)
        # Alg. 1 step 10: gbest state from its owner
        owner = runner.owner_of(out.gbest_particle)
        if runner.rank == owner:
            self.engine.gbest_state(self.Ua[0], self.cen[0])
        if self.dist is not None and runner.world > 1:
            broadcast_(self.dist, self.Ua, owner)
            broadcast_(self.dist, self.cen, owner)
        ev[3].record()
        # Alg. 1 step 11: final IFCM at (lambda*, xi*) until eps, then argmax
        lx = torch.tensor([[out.lam, out.xi]], dtype=torch.float64, device=self.dev)
        if self.shard_final:
            sl = self.slab
            sl.load_x(x)
            sl.load_state(self.Ua, self.cen)
            sl.run(lx, cfg.max_iter, eps=cfg.eps)
            self.cen.copy_(sl.centers)
            loc = ctx.argmax(sl.local_U()[0], nx, ny, sl.nz, cfg.C)
            labels = self._gather_labels(loc)
            final_iters = int(sl.stats[0, 2].item())
        else:
            stats.zero_()
            # canonical=True: pifcm_iterate_ex takes the pointwise FCM step at
            # lambda = xi = 0 itself, exactly as pifcm_segment's final IFCM
            ctx.iterate(x, self.Ua, self.Ub, self.cen, lx, cfg, iters=cfg.max_iter, stats=stats, nx=nx,
                        canonical=True)
            labels = ctx.argmax(self.Ub[0], nx, ny, nz, cfg.C)
            final_iters = int(stats[0, 2].item())
        ev[4].record()
        torch.cuda.synchronize()
        self.labels = labels
        return {"lambda": out.lam, "xi": out.xi, "J": out.J, "generations": out.generations,
                "gbest_particle": out.gbest_particle, "fcm_iters": fcm_iters,
                "final_iters": final_iters, "centers": self.cen[0, :cfg.C].tolist(),
                "t_norm": ev[0].elapsed_time(ev[1]) * 1e-3, "t_init": ev[1].elapsed_time(ev[2]) * 1e-3,
                "t_pso": ev[2].elapsed_time(ev[3]) * 1e-3, "t_final": ev[3].elapsed_time(ev[4]) * 1e-3,
                "t_total": ev[0].elapsed_time(ev[4]) * 1e-3}

    def _gather_labels(self, loc: torch.Tensor) -> torch.Tensor:
        sl = self.slab
        if sl.world == 1:
            return loc
        d = sl.dist
        self.lab_pad[sl.rank, : loc.numel()] = loc.view(-1)
        src = _coll_tensor(d, self.lab_pad[sl.rank].contiguous())
        out = _coll_tensor(d, self.lab_pad)
        if src.device.type == "cpu":
            torch.cuda.current_stream().synchronize()
        d.all_gather_into_tensor(out.view(-1), src)
        if out is not self.lab_pad:
            self.lab_pad.copy_(out)
        return torch.cat([self.lab_pad[r, :n] for r, n in enumerate(self.lab_counts)]).view(
            self.nz, self.ny, self.nx)

    def segment_host(self, vol_host: torch.Tensor, labels_host: torch.Tensor) -> dict:
        """Host (pinned) u8 volume in, host labels out (H2D / D2H inside)."""
        vol = vol_host.to(self.dev, non_blocking=True)
        rep = self.segment(vol)
        labels_host.copy_(self.labels, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return rep


# ----------------------------------------------------------------------------
# z-slab sharding (volumes too large for one GPU: SURVEY 8(e), the C5 workload)
def slab_range(nz_total: int, world: int, rank: int, tz: int) -> tuple[int, int]:
    """(z0, nz) of rank's slab: whole tz-plane global chunks (tz =
    pifcm_slab_chunk of the volume), split as evenly as possible."""
    chunks = -(-nz_total // tz)
    c0, c1 = shard_range(chunks, world, rank)
    z0 = c0 * tz
    return z0, min(c1 * tz, nz_total) - z0


def _coll_tensor(dist, t):
    return t.cpu() if dist.get_backend() == "gloo" and t.device.type == "cuda" else t


def _halo_sendrecv(dist, rank, world, send_lo, send_hi, recv_lo, recv_hi):
    """Boundary planes to / from the neighbouring slabs (one batched send/recv;
    gloo carries CUDA tensors through host copies)."""
    ops = []
    if rank > 0:
        ops += [("send", send_lo, rank - 1), ("recv", recv_lo, rank - 1)]
    if rank < world - 1:
        ops += [("send", send_hi, rank + 1), ("recv", recv_hi, rank + 1)]
    if not ops:
        return
    if dist.get_backend() == "gloo" and any(t.device.type == "cuda" for _, t, _ in ops):
        torch.cuda.current_stream().synchronize()
    bufs = [(k, _coll_tensor(dist, t), t, peer) for k, t, peer in ops]
    reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend if k == "send" else dist.irecv, b, peer)
                                   for k, b, _, peer in bufs])
    for r in reqs:
        r.wait()
    for k, b, t, _ in bufs:
        if k == "recv" and b is not t:
            t.copy_(b)


class _SlabGeometry:
    """This rank's slab of a volume and the record bookkeeping shared by the
    slab drivers: global chunk size, slab grid, per-rank record counts, the
    local / padded / gathered record buffers and their all-gather."""

    def __init__(self, ctx, nx, ny, nz_total, P, dist, H=1):
        """H: halo planes per side of the slab arrays (the cfg's v)."""
        from .api import _grid
        self.ctx, self.dist, self.P, self.H = ctx, dist, P, H
        self.world = dist.get_world_size() if dist is not None else 1
        self.rank = dist.get_rank() if dist is not None else 0
        self.nx, self.ny, self.nz_total = nx, ny, nz_total
        self.tz = ctx.slab_chunk(nx, ny, nz_total)
        self.z0, self.nz = slab_range(nz_total, self.world, self.rank, self.tz)
        self.grid = _grid(nx, ny, self.nz, z0=self.z0, nz_total=nz_total)
        self.plane = nx * ny
        nrecs = []
        for r in range(self.world):
            z0, nz = slab_range(nz_total, self.world, r, self.tz)
            nrecs.append(ctx.slab_records(_grid(nx, ny, nz, z0=z0, nz_total=nz_total)))
        self.nrec = nrecs[self.rank]
        self.nrec_max = max(nrecs)
        self.dev = getattr(ctx, "torch_device", None) or torch.device(f"cuda:{ctx.device}")
        self.counts = torch.tensor(nrecs, dtype=torch.int32, device=self.dev)
        self.rec = torch.zeros((P, self.nrec, 10), dtype=torch.float64, device=self.dev)
        self.rec_pad = torch.zeros((P, self.nrec_max, 10), dtype=torch.float64, device=self.dev)
        self.gathered = torch.zeros((self.world, P, self.nrec_max, 10), dtype=torch.float64, device=self.dev)
        self.halo = {k: torch.zeros((P, H * self.plane, 4), dtype=torch.float32, device=self.dev)
                     for k in ("send_lo", "send_hi", "recv_lo", "recv_hi")}

    def gather_records(self) -> torch.Tensor:
        """Records of every rank in rank order, [world][P][nrec_max][10]."""
        self.rec_pad[:, : self.nrec] = self.rec
        if self.world == 1:
            return self.rec_pad
        d = self.dist
        src = _coll_tensor(d, self.rec_pad)
        out = _coll_tensor(d, self.gathered)
        if src is not self.rec_pad:
            torch.cuda.current_stream().synchronize()
        d.all_gather_into_tensor(out.view(self.world * self.P, self.nrec_max, 10), src)
        if out is not self.gathered:
            self.gathered.copy_(out)
        return self.gathered

    def exchange(self, pack, unpack):
        """pack(op, buf) fills buf with the H boundary planes op (0 lower, 1 upper);
        unpack(op, buf or None) writes the halo (2 lower, 3 upper; None at the
        volume ends = zero fill)."""
        h = self.halo
        if self.world > 1:
            if self.rank > 0:
                pack(0, h["send_lo"])
            if self.rank < self.world - 1:
                pack(1, h["send_hi"])
            _halo_sendrecv(self.dist, self.rank, self.world, h["send_lo"], h["send_hi"], h["recv_lo"],
                           h["recv_hi"])
        unpack(2, h["recv_lo"] if self.rank > 0 else None)
        unpack(3, h["recv_hi"] if self.rank < self.world - 1 else None)

    def slab_planes(self, t: torch.Tensor) -> torch.Tensor:
        """Planes [z0 - H, z0 + nz + H) of a full-volume [nz_total][...] tensor,
        zero where they fall outside the volume."""
        H = self.H
        out = torch.zeros((self.nz + 2 * H,) + tuple(t.shape[1:]), dtype=t.dtype, device=self.dev)
        lo, hi = max(self.z0 - H, 0), min(self.z0 + self.nz + H, self.nz_total)
        out[lo - (self.z0 - H): hi - (self.z0 - H)] = t[lo:hi].to(self.dev)
        return out


class SlabIfcm:
    """Jacobi IFCM iterations of P states over a volume split into z-slabs, one
    per rank.  Per iteration: halo exchange of one U plane per neighbour and
    state (pack / unpack kernels, send / recv), pifcm_slab_step on the local
    planes, an all-gather of the per-chunk partial records, pifcm_slab_finalize
    (Eq. 3 / Eq. 1 in global chunk order: identical on every rank and for any
    number of slabs)."""

    def __init__(self, ctx, cfg, nx, ny, nz_total, P, dist=None):
        self.ctx, self.cfg, self.P, self.dist = ctx, cfg, P, dist
        self.H = H = cfg.v  # halo planes per side (Eq. 9 radius in z)
        self.geo = _SlabGeometry(ctx, nx, ny, nz_total, P, dist, H)
        g = self.geo
        self.world, self.rank, self.tz = g.world, g.rank, g.tz
        self.nx, self.ny, self.nz_total = nx, ny, nz_total
        self.z0, self.nz, self.grid, self.plane = g.z0, g.nz, g.grid, g.plane
        self.dev = g.dev
        self.Ua = torch.zeros((P, (self.nz + 2 * H) * self.plane, 4), dtype=torch.float32, device=self.dev)
        self.Ub = torch.zeros_like(self.Ua)
        self.centers = torch.zeros((P, 4), dtype=torch.float32, device=self.dev)
        self.stats = torch.zeros((P, 4), dtype=torch.float64, device=self.dev)
        self.swaps = 0

    # -- data in / out
    def load_x(self, x_full: torch.Tensor):
        """x_full [nz_total][ny][pitch] (any device) -> the slab with its halo
        planes (zero outside the volume)."""
        self.x = self.geo.slab_planes(x_full)
        return self.x

    def set_x(self, x_slab: torch.Tensor):
        """x of the slab's arrays [nz + 2H][ny][pitch] (halo planes included)."""
        self.x = x_slab

    def load_state(self, U_full: torch.Tensor, centers: torch.Tensor):
        """U_full [P][nz_total*ny*nx][4]: this slab's planes (halos exchanged later)."""
        pl, H = self.plane, self.H
        self.Ua[:, H * pl: pl * (self.nz + H)] = U_full[:, self.z0 * pl:(self.z0 + self.nz) * pl].to(self.dev)
        self.centers.copy_(centers.view(self.P, 4))
        self.stats.zero_()
        self.swaps = 0

    def load_local(self, U_slab: torch.Tensor, centers: torch.Tensor):
        """U_slab [P][(nz+2H)*ny*nx][4] already in the slab layout."""
        self.Ua.copy_(U_slab.view_as(self.Ua))
        self.centers.copy_(centers.view(self.P, 4))
        self.stats.zero_()
        self.swaps = 0

    def local_U(self) -> torch.Tensor:
        return self.Ua[:, self.H * self.plane: self.plane * (self.nz + self.H)]

    # -- one iteration
    def exchange(self, U):
        ctx, g, P, H = self.ctx, self.grid, self.P, self.H
        self.geo.exchange(lambda op, buf: ctx.slab_halo(g, P, op, U, buf, v=H),
                          lambda op, buf: ctx.slab_halo(g, P, op, U, buf, v=H))

    def step(self, lam_xi: torch.Tensor, eps: float = 0.0):
        """One iteration (no host synchronisation).  A converged state is
        skipped by the step kernel, so its latest U stays in the buffer its
        last real step wrote: sync_states() moves it back into Ua."""
        self.exchange(self.Ua)
        self.ctx.slab_step(self.grid, self.cfg, self.x, self.Ua, self.Ub, self.centers, lam_xi, self.geo.rec,
                           stats=self.stats)
        recs = self.geo.gather_records()
        self.ctx.slab_finalize(self.cfg.C, self.P, self.world, self.geo.nrec_max, recs, self.centers,
                               stats=self.stats, eps=eps, counts=self.geo.counts)
        self.Ua, self.Ub = self.Ub, self.Ua
        self.swaps += 1

    def sync_states(self):
        """After steps that skipped converged states: state p's latest U was
        written by its stats[p, 2]-th step, into the buffer that was current
        after that many swaps; copy it into Ua where that is the other one."""
        done = self.stats[:, 2].to(torch.int64).cpu()
        for p in range(self.P):
            if (int(done[p]) - self.swaps) % 2:
                self.Ua[p].copy_(self.Ub[p])

    def run(self, lam_xi: torch.Tensor, iters: int, eps: float = 0.0, check_every: int = 4) -> int:
        """`iters` iterations from the current states (stats restart)."""
        self.stats.zero_()
        self.swaps = 0
        done = 0
        for it in range(iters):
            self.step(lam_xi, eps)
            done = it + 1
            if eps > 0 and (it + 1) % check_every == 0 and bool((self.stats[:, 3] != 0).all()):
                break
        self.sync_states()
        return done


class _DevArray:
    """A raw device allocation seen by torch (__cuda_array_interface__)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _as_tensor(ptr, shape, dtype, dev):
    typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4"}[dtype]
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device=dev)


class SlabIfcmP2P:
    """SlabIfcm with the exchange done by the GPUs over peer memory
    (pifcm_slab_p2p_run): every rank maps the others' state buffers,
    gathered-record buffers and flag words (CUDA IPC handles swapped once
    through torch.distributed); per iteration the step, a put kernel that
    stores the boundary planes into the neighbours' halo planes and the
    records into every rank's gathered buffer, a device barrier and the
    canonical finalisation -- no NCCL call and no host round trip between the
    convergence checks.  Results are bit-identical to SlabIfcm."""

    def __init__(self, ctx, cfg, nx, ny, nz_total, P, dist=None):
        from . import _abi
        self.ctx, self.cfg, self.P, self.dist = ctx, cfg, P, dist
        self.H = H = cfg.v  # halo planes per side
        self.geo = g = _SlabGeometry(ctx, nx, ny, nz_total, P, dist, H)
        self.world, self.rank, self.nz, self.grid, self.plane = g.world, g.rank, g.nz, g.grid, g.plane
        if self.world > _abi.MAX_PEERS:
            raise RuntimeError(f"peer exchange supports at most {_abi.MAX_PEERS} ranks")
        self.dev = g.dev
        sb = P * (self.nz + 2 * H) * self.plane * 16
        rb = self.world * P * g.nrec_max * 10 * 8
        # every step below is agreed on by all ranks, so that either all of
        # them use peer memory or none does (a rank that cannot map a peer
        # must not leave the others waiting at a barrier)
        self._own, self._opened = [], []
        ok = 1
        try:
            for nb in (sb, sb, rb, rb, 4 * (self.world + 2)):
                self._own.append(ctx.peer_alloc(nb))
            mine = ([ctx.peer_handle(p) for p in self._own], self.nz)
        except Exception:
            ok, mine = 0, None
        allh = [mine]
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, mine)
        ok = ok and all(h is not None for h in allh)
        ptrs = []
        if ok:
            try:
                for w, (hs, _) in enumerate(allh):
                    if w == self.rank:
                        ptrs.append(self._own)
                    else:
                        op = [ctx.peer_open(h) for h in hs]
                        self._opened += op
                        ptrs.append(op)
            except Exception:
                ok = 0
        if self.world > 1:
            flag = torch.tensor([ok], dtype=torch.int32,
                                device=self.dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ok = int(flag.item())
        if not ok:
            for p in self._opened:
                ctx.peer_close(p)
            for p in self._own:
                ctx.peer_free(p)
            raise RuntimeError("peer memory mapping is not available on every rank")
        pe = _abi.Peers()
        pe.world, pe.rank = self.world, self.rank
        for w in range(self.world):
            pe.U[0][w], pe.U[1][w], pe.rec[0][w], pe.rec[1][w], pe.flags[w] = ptrs[w]
            pe.nz[w] = allh[w][1]
        self.peers = pe
        shape = (P, (self.nz + 2 * H) * self.plane, 4)
        self.U = [_as_tensor(self._own[i], shape, torch.float32, self.dev) for i in range(2)]
        self.centers = torch.zeros((P, 4), dtype=torch.float32, device=self.dev)
        self.stats = torch.zeros((P, 4), dtype=torch.float64, device=self.dev)
        self.epoch, self.cur = 0, 0
        if self.world > 1:
            dist.barrier()  # every mapping is open before any rank writes into it

    def close(self):
        for p in self._opened:
            self.ctx.peer_close(p)
        if self.world > 1:
            self.dist.barrier()  # nobody maps this rank's memory any more
        for p in self._own:
            self.ctx.peer_free(p)
        self._opened, self._own = [], []

    def load_x(self, x_full: torch.Tensor):
        self.x = self.geo.slab_planes(x_full)
        return self.x

    def set_x(self, x_slab: torch.Tensor):
        self.x = x_slab

    def load_state(self, U_full: torch.Tensor, centers: torch.Tensor):
        """U_full [P][nz_total*ny*nx][4]: this slab's local planes (the outer
        halo planes stay zero, the interior ones are exchanged by the run)."""
        pl, H = self.plane, self.H
        self.U[self.cur][:, H * pl: pl * (self.nz + H)] = U_full[:, self.geo.z0 * pl:(self.geo.z0 + self.nz) * pl]
        self.centers.copy_(centers.view(self.P, 4))

    def load_local(self, U_slab: torch.Tensor, centers: torch.Tensor):
        """U_slab [P][(nz+2H)*ny*nx][4] in the slab layout (local planes used)."""
        pl, H = self.plane, self.H
        self.U[self.cur][:, H * pl: pl * (self.nz + H)] = U_slab.view(self.P, -1, 4)[:, H * pl: pl * (self.nz + H)]
        self.centers.copy_(centers.view(self.P, 4))

    def local_U(self) -> torch.Tensor:
        return self.U[self.cur][:, self.H * self.plane: self.plane * (self.nz + self.H)]

    @property
    def Ua(self) -> torch.Tensor:
        """The current states in the slab layout (as SlabIfcm.Ua)."""
        return self.U[self.cur]

    def run(self, lam_xi: torch.Tensor, iters: int, eps: float = 0.0) -> int:
        from dataclasses import replace
        cfg = replace(self.cfg, eps=eps)
        start = self.cur
        self.epoch, self.cur, done = self.ctx.slab_p2p_run(
            self.grid, cfg, self.x, self.peers, self.P, self.geo.counts, self.geo.nrec_max, self.centers,
            lam_xi, self.stats, self.geo.rec, iters, self.epoch, self.cur)
        # a converged state was skipped from then on: its latest U is in the
        # buffer its last real step wrote
        n = self.stats[:, 2].to(torch.int64).cpu()
        for p in range(self.P):
            b = (start + int(n[p])) % 2
            if b != self.cur:
                self.U[self.cur][p].copy_(self.U[b][p])
        return done


class SlabPso:
    """Alg. 1 steps 3-10 over z-slab ranks (pifcm_slab_pso_*): every rank holds
    all P particles' states for its slab and the identical swarm; per
    generation a halo exchange of every particle's current state, the slab
    step of all particles, an all-gather of their records, the fitness /
    centres finalisation and the device PSO update -- the same on every rank,
    so fitness vectors and trajectories are bit-identical for any number of
    slabs."""

    def __init__(self, ctx, cfg, pso, nx, ny, nz_total, dist=None, check_every: int = 4):
        from dataclasses import replace
        self.ctx, self.cfg, self.dist = ctx, cfg, dist
        self.pso = replace(pso, p_begin=0, p_end=0)
        self.geo = _SlabGeometry(ctx, nx, ny, nz_total, pso.P, dist, cfg.v)
        self.grid = self.geo.grid
        self.ws = ctx.slab_workspace(self.grid, cfg, self.pso)
        self.check_every = check_every

    def init(self, U0_slab: torch.Tensor, c0: torch.Tensor):
        """U0_slab [(nz+2v)*ny*nx][4] (slab layout), c0 [4]."""
        self.ctx.slab_pso_init(self.grid, self.cfg, self.pso, U0_slab, c0, self.ws)

    def generation(self, x_slab: torch.Tensor):
        c, g, cfg, pso, ws = self.ctx, self.grid, self.cfg, self.pso, self.ws
        self.geo.exchange(lambda op, buf: c.slab_pso_halo(g, cfg, pso, ws, op, buf),
                          lambda op, buf: c.slab_pso_halo(g, cfg, pso, ws, op, buf))
        c.slab_pso_eval(g, cfg, pso, x_slab, ws, self.geo.rec)
        recs = self.geo.gather_records()
        c.slab_pso_finalize(g, cfg, pso, ws, self.geo.world, self.geo.nrec_max, recs, counts=self.geo.counts)
        c.slab_pso_update(g, cfg, pso, ws)

    def fitness(self) -> torch.Tensor:
        return self.ctx.slab_pso_fitness(self.grid, self.cfg, self.pso, self.ws)

    def run(self, x_slab: torch.Tensor, max_gen: int, early_stop: bool, trace=None) -> PsoOutcome:
        for gen in range(max_gen):
            self.generation(x_slab)
            if trace is not None:
                trace.append(self.fitness().cpu().clone())
            if early_stop and (gen + 1) % self.check_every == 0:
                _, stopped = self.ctx.slab_pso_result(self.grid, self.cfg, self.pso, self.ws)
                if stopped:
                    break
        s, _ = self.ctx.slab_pso_result(self.grid, self.cfg, self.pso, self.ws)
        return PsoOutcome(s.lam, s.xi, s.J, s.generations, s.gbest_particle)

    def gbest_state(self, U_out: torch.Tensor, c_out: torch.Tensor):
        """The gbest particle's slab state (every rank holds its own part)."""
        self.ctx.slab_pso_gbest_state(self.grid, self.cfg, self.pso, self.ws, U_out, c_out)


class SlabSegmenter:
    """The whole method (Alg. 1 / Alg. 2) on a volume split into z-slabs, one
    per rank: global min-max (all-reduce) and histogram (all-reduce) for the
    GMM start, the FCM start (lambda = xi = 0) as slab iterations, the PSO
    over slabs (SlabPso), the final IFCM over slabs (SlabIfcm) and the argmax
    of each slab, gathered.  Every reduction is over global z-chunk records in
    a fixed order, so all results are bit-identical for any number of ranks."""

    def __init__(self, ctx, cfg, pso, shape, dist=None):
        self.ctx, self.cfg, self.pso, self.dist = ctx, cfg, pso, dist
        self.nz, self.ny, self.nx = shape
        self.ifcm = _slab_driver(ctx, cfg, self.nx, self.ny, self.nz, 1, dist)
        self.swarm = SlabPso(ctx, cfg, pso, self.nx, self.ny, self.nz, dist)
        self.geo = self.ifcm.geo
        self.dev = self.geo.dev
        g = self.geo
        self.lab_counts = [slab_range(self.nz, g.world, r, g.tz)[1] * self.nx * self.ny for r in range(g.world)]
        self.lab_pad = torch.zeros((g.world, max(self.lab_counts)), dtype=torch.uint8, device=self.dev)
        self.keep_trace = False  # record every generation's fitness vector (host sync per generation)
        self.trace = None

    def _allreduce(self, t, op):
        if self.geo.world == 1:
            return t
        d = self.dist
        h = _coll_tensor(d, t)
        d.all_reduce(h, op=op)
        if h is not t:
            t.copy_(h)
        return t

    def segment(self, vol: torch.Tensor) -> dict:
        """vol: the whole u8 volume [nz][ny][nx] (any device); each rank reads
        its slab planes."""
        ctx, cfg, g, d = self.ctx, self.cfg, self.geo, self.dist
        if vol.dtype != torch.uint8:
            raise TypeError("the z-slab pipeline takes uint8 volumes")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        # Alg. 2 step 1: global min-max (all-reduce) and the R15 histogram
        H = g.H
        v = g.slab_planes(vol)                      # [nz+2H][ny][nx], zero outside the volume
        own = v[H: g.nz + H]
        mm = torch.zeros(2, dtype=torch.int32, device=self.dev)
        ctx.minmax_u8(own, mm)
        if g.world > 1:
            lo, hi = mm[:1].clone(), mm[1:].clone()
            self._allreduce(lo, d.ReduceOp.MIN)
            self._allreduce(hi, d.ReduceOp.MAX)
            mm = torch.cat([lo, hi])
        x = ctx.normalize_u8_range(v, mm)
        # halo planes outside the volume stay zero (normalising the zero
        # padding would give them the value of intensity 0)
        lo_out = max(0, H - g.z0)
        hi_out = max(0, g.z0 + g.nz + H - g.nz_total)
        if lo_out:
            x[:lo_out].zero_()
        if hi_out:
            x[g.nz + 2 * H - hi_out:].zero_()
        hist = ctx.hist_u8(own, mm)
        if g.world > 1:
            self._allreduce(hist, d.ReduceOp.SUM)
        c0 = ctx.gmm_init(hist, cfg.C)
        ev[1].record()
        # Alg. 1 step 2: FCM start on the global value histogram (R24): the
        # ranks' counts are summed, every rank runs the identical FCM loop and
        # writes the memberships of its own planes (halo planes zero; the PSO
        # exchanges them)
        sl = self.ifcm
        sl.set_x(x)
        counts = ctx.value_hist(own)
        if g.world > 1:
            self._allreduce(counts, d.ReduceOp.SUM)
        c_prev, c_fcm, fst = ctx.fcm_hist(counts, mm, c0, cfg)
        pl = self.nx * self.ny
        U0 = sl.Ua[0]
        U0[:H * pl].zero_()
        U0[pl * (g.nz + H):].zero_()
        ctx.fcm_memberships(x[H: g.nz + H], c_prev, cfg.C, cfg.m, self.nx, U=U0[H * pl: pl * (g.nz + H)])
        fcm_iters = int(fst[2].item())
        ev[2].record()
        # Alg. 1 steps 3-10: PSO over slabs from (U_fcm, c_fcm)
        sw = self.swarm
        sw.init(sl.Ua[0], c_fcm)
        self.trace = [] if self.keep_trace else None
        out = sw.run(x, self.pso.max_gen, early_stop=self.pso.patience > 0, trace=self.trace)
        Ug = torch.empty_like(sl.Ua[0])
        cg = torch.empty(4, dtype=torch.float32, device=self.dev)
        sw.gbest_state(Ug, cg)
        ev[3].record()
        # Alg. 1 step 11: final IFCM at (lambda*, xi*), then argmax of each slab
        lx = torch.tensor([[out.lam, out.xi]], dtype=torch.float64, device=self.dev)
        sl.load_local(Ug.unsqueeze(0), cg.view(1, 4))
        sl.run(lx, cfg.max_iter, eps=cfg.eps)
        final_iters = int(sl.stats[0, 2].item())
        loc = ctx.argmax(sl.local_U()[0], self.nx, self.ny, g.nz, cfg.C)
        self.labels = self._gather_labels(loc)
        ev[4].record()
        torch.cuda.synchronize()
        return {"lambda": out.lam, "xi": out.xi, "J": out.J, "generations": out.generations,
                "gbest_particle": out.gbest_particle, "fcm_iters": fcm_iters, "final_iters": final_iters,
                "c_init": c0[: cfg.C].tolist(), "centers": sl.centers[0, : cfg.C].tolist(),
                "t_norm": ev[0].elapsed_time(ev[1]) * 1e-3, "t_init": ev[1].elapsed_time(ev[2]) * 1e-3,
                "t_pso": ev[2].elapsed_time(ev[3]) * 1e-3, "t_final": ev[3].elapsed_time(ev[4]) * 1e-3,
                "t_total": ev[0].elapsed_time(ev[4]) * 1e-3}

    def _gather_labels(self, loc: torch.Tensor) -> torch.Tensor:
        g = self.geo
        if g.world == 1:
            return loc
        d = self.dist
        self.lab_pad[g.rank, : loc.numel()] = loc.reshape(-1)
        src = _coll_tensor(d, self.lab_pad[g.rank].contiguous())
        out = _coll_tensor(d, self.lab_pad)
        if src.device.type == "cpu":
            torch.cuda.current_stream().synchronize()
        d.all_gather_into_tensor(out.view(-1), src)
        if out is not self.lab_pad:
            self.lab_pad.copy_(out)
        return torch.cat([self.lab_pad[r, :n] for r, n in enumerate(self.lab_counts)]).view(
            self.nz, self.ny, self.nx)
