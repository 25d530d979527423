"""Python binding of libpifcm.so: the same calls as include/pifcm.h, taking
torch tensors (device memory) and doing argument marshalling only.  Every
step of the method runs in the library's CUDA kernels; torch provides device
memory and streams.

Citations: PAPER:N = line N of the paper text; Rk = DESIGN.md reading k.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import torch

from . import _abi

__all__ = ["IfcmConfig", "PsoConfig", "PifcmError", "Context", "pitch_of", "to_pitched_x",
           "to_aos", "from_aos"]


class PifcmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_abi.STATUS.get(code, code)}: {msg}")
        self.code = code


@dataclass
class IfcmConfig:
    """Alg. 1 inputs c, v, h, m, epsilon + reading R1 (q_mode)."""
    C: int = 4
    m: float = 2.0
    v: int = 1
    h: float = 1.0
    q_mode: int = _abi.Q_LITERAL
    eps: float = 1e-5
    max_iter: int = 100

    def c(self) -> _abi.IfcmCfg:
        return _abi.IfcmCfg(self.C, self.m, self.v, self.h, self.q_mode, self.eps, self.max_iter)


@dataclass
class PsoConfig:
    """Alg. 1 steps 3-9, reading R12."""
    P: int = 32
    ring_k: int = 1
    max_gen: int = 30
    patience: int = 3
    tol: float = 1e-4
    v0: float = 0.1
    vmax: float = 0.5
    seed: int = 12345
    p_begin: int = 0
    p_end: int = 0
    fitness: int = 0  # 0 CHAINED (R11), 1 ANCHORED, 2 LEADER (R22)
    eval_batch: int = 0  # CHAINED: states per evaluation launch (0 = all; fewer slots otherwise)

    def c(self) -> _abi.PsoCfg:
        return _abi.PsoCfg(self.P, self.ring_k, self.max_gen, self.patience, self.tol, self.v0,
                           self.vmax, self.seed, self.fitness, self.p_begin, self.p_end, self.eval_batch)


def dtype_code(vol: torch.Tensor) -> int:
    """pifcm_dtype of a volume tensor (u8, uint16, float32)."""
    codes = {torch.uint8: _abi.U8, torch.uint16: _abi.U16, torch.float32: _abi.F32}
    if vol.dtype not in codes:
        raise TypeError(f"volumes are uint8, uint16 or float32, not {vol.dtype}")
    return codes[vol.dtype]


def pitch_of(nx: int) -> int:
    return (nx + 3) // 4 * 4


def to_pitched_x(x, device) -> torch.Tensor:
    """[nz, ny, nx] intensities -> device fp32 [nz, ny, pitch] (zero padded)."""
    x = torch.as_tensor(x, dtype=torch.float32)
    nz, ny, nx = x.shape
    out = torch.zeros((nz, ny, pitch_of(nx)), dtype=torch.float32, device=device)
    out[:, :, :nx] = x.to(device)
    return out


def to_aos(U, device) -> torch.Tensor:
    """[..., N, C] memberships -> device fp32 [..., N, 4] (AoS-C4, zero padded)."""
    U = torch.as_tensor(U, dtype=torch.float32)
    shape = list(U.shape)
    C = shape[-1]
    shape[-1] = 4
    out = torch.zeros(shape, dtype=torch.float32, device=device)
    out[..., :C] = U.to(device)
    return out


def from_aos(U: torch.Tensor, C: int) -> torch.Tensor:
    return U[..., :C]


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream or None


def _grid(nx, ny, nz, pitch=None, z0=0, nz_total=0) -> _abi.Grid:
    return _abi.Grid(nx, ny, nz, pitch if pitch is not None else pitch_of(nx), z0, nz_total)


@dataclass
class PsoSummary:
    lam: float
    xi: float
    J: float
    generations: int
    gbest_particle: int
    centers: list = field(default_factory=list)


class Context:
    """Owns a pifcm_ctx on one CUDA device."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("pifcm needs a CUDA device (no CPU fallback)")
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = int(device)
        self.lib = _abi.load()
        h = ct.c_void_p()
        torch.cuda.init()
        with torch.cuda.device(self.device):
            rc = self.lib.pifcm_ctx_create(self.device, ct.byref(h))
        if rc != 0:
            raise PifcmError(rc, "pifcm_ctx_create failed")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self.lib.pifcm_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc: int):
        if rc != 0:
            raise PifcmError(rc, self.lib.pifcm_last_error(self._h).decode())

    # ------------------------------------------------------------ multi-process
    def attach_dist(self, rank: int, world: int, pg=None, backend: str = "nccl"):
        """pifcm_ctx_dist: give this context a communicator for the
        particle-sharded pifcm_segment.  backend "nccl": NCCL inside the
        library (rank 0's pifcm_nccl_unique_id is shared through the
        torch.distributed process group `pg`); "host": the library calls back
        into torch.distributed (gloo) with host buffers -- ranks sharing a GPU.
        world == 1 detaches."""
        import torch.distributed as tdist
        d = _abi.Dist(rank, world, None, 0)
        coll = None
        if world > 1 and backend == "nccl":
            uid = (ct.c_uint8 * 128)()
            if rank == 0:
                rc = self.lib.pifcm_nccl_unique_id(uid)
                if rc != 0:
                    raise PifcmError(rc, "pifcm_nccl_unique_id failed")
            obj = [bytes(uid)]
            tdist.broadcast_object_list(obj, src=0, group=pg)
            uid = (ct.c_uint8 * 128).from_buffer_copy(obj[0])
            self._uid = uid
            d.nccl_unique_id = ct.cast(uid, ct.c_void_p)
        elif world > 1:
            def _ag(user, src, dst, n):
                try:
                    t = torch.frombuffer(bytearray(ct.string_at(src, n)), dtype=torch.uint8)
                    out = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
                    tdist.all_gather(out, t, group=pg)
                    cat = torch.cat(out).numpy()  # (kept alive across the copy)
                    ct.memmove(dst, cat.ctypes.data, n * world)
                    return 0
                except Exception:
                    return 1

            def _bc(user, buf, n, root):
                try:
                    t = torch.frombuffer(bytearray(ct.string_at(buf, n)), dtype=torch.uint8)
                    tdist.broadcast(t, src=root, group=pg)
                    arr = t.numpy()
                    ct.memmove(buf, arr.ctypes.data, n)
                    return 0
                except Exception:
                    return 1

            coll = _abi.HostColl(None, _abi.HOST_ALLGATHER(_ag), _abi.HOST_BROADCAST(_bc))
            self._coll = coll  # keep the callbacks alive
        self._ck(self.lib.pifcm_ctx_dist(self._h, ct.byref(d), ct.byref(coll) if coll is not None else None))
        self.rank, self.world = rank, world

    def dist_range(self, P: int, world: int, rank: int) -> tuple[int, int]:
        a, b = ct.c_int32(), ct.c_int32()
        self._ck(self.lib.pifcm_dist_range(P, world, rank, ct.byref(a), ct.byref(b)))
        return a.value, b.value

    def launch_count(self) -> int:
        return int(self.lib.pifcm_launch_count(self._h))

    def timing_enable(self, on: bool = True):
        self._ck(self.lib.pifcm_timing_enable(self._h, 1 if on else 0))

    def timing_read(self, batched: bool = True):
        """-> (summed fused-step kernel ms, launches, algorithmic bytes) of the
        batched (P > 1, PSO generations) or single-state launches."""
        ms, n, b = ct.c_double(), ct.c_int64(), ct.c_double()
        self._ck(self.lib.pifcm_timing_read(self._h, 1 if batched else 0, ct.byref(ms), ct.byref(n),
                                            ct.byref(b)))
        return ms.value, n.value, b.value

    # ------------------------------------------------------------ workspace
    def workspace_size(self, nx, ny, nz, cfg: IfcmConfig, pso: PsoConfig | None) -> int:
        n = ct.c_size_t()
        g = _grid(nx, ny, nz)
        rc = self.lib.pifcm_workspace_size(ct.byref(g), ct.byref(cfg.c()),
                                           ct.byref(pso.c()) if pso else None, ct.byref(n))
        self._ck(rc)
        return n.value

    def workspace(self, nx, ny, nz, cfg: IfcmConfig, pso: PsoConfig | None) -> torch.Tensor:
        return torch.empty(self.workspace_size(nx, ny, nz, cfg, pso), dtype=torch.uint8,
                           device=f"cuda:{self.device}")

    # ------------------------------------------------------------ iterate
    def iterate(self, x: torch.Tensor, U_in: torch.Tensor, U_out: torch.Tensor,
                centers: torch.Tensor, lam_xi: torch.Tensor, cfg: IfcmConfig, iters: int = 1,
                stats: torch.Tensor | None = None, nx: int | None = None, stream=None,
                canonical: bool = False, per_step: bool = False):
        """pifcm_iterate(_ex): x [nz,ny,pitch] f32; U_in/U_out [P,nz*ny*nx,4] f32;
        centers [P,4] f32; lam_xi [P,2] f64; stats [P,4] f64 or None.
        canonical: the z-chunk decomposition of pifcm_segment's final IFCM.
        per_step: one launch per iteration (no cooperative 2D loop)."""
        nz, ny, pitch = x.shape
        P = U_in.shape[0]
        if nx is None:
            nx = U_in.shape[1] // (ny * nz)
        g = _grid(nx, ny, nz, pitch)
        n = ct.c_size_t()
        self._ck(self.lib.pifcm_iterate_workspace_size(ct.byref(g), ct.byref(cfg.c()), P, iters,
                                                       ct.byref(n)))
        ws = torch.empty(max(n.value, 1), dtype=torch.uint8, device=x.device)
        rc = self.lib.pifcm_iterate_ex(self._h, ct.byref(g), ct.byref(cfg.c()), _ptr(x), _ptr(U_in),
                                       _ptr(U_out), _ptr(centers), _ptr(lam_xi), P, iters, _ptr(stats),
                                       _ptr(ws), n.value,
                                       (_abi.ITER_CANONICAL if canonical else 0) | (_abi.ITER_PER_STEP if per_step else 0),
                                       _stream(stream))
        self._ck(rc)
        return U_out

    # ------------------------------------------------------------ PSO
    def pso_init(self, grid, cfg, pso, U0, c0, ws, stream=None):
        self._ck(self.lib.pifcm_pso_init(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                         _ptr(U0), _ptr(c0), _ptr(ws), ws.numel(), _stream(stream)))

    def pso_eval(self, grid, cfg, pso, x, ws, stream=None):
        self._ck(self.lib.pifcm_pso_eval(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                         _ptr(x), _ptr(ws), ws.numel(), _stream(stream)))

    def pso_update(self, grid, cfg, pso, ws, x=None, stream=None):
        """x: required for the ANCHORED / LEADER fitness modes."""
        self._ck(self.lib.pifcm_pso_update(self._h, ct.byref(grid), ct.byref(cfg.c()),
                                           ct.byref(pso.c()), _ptr(x), _ptr(ws), ws.numel(), _stream(stream)))

    def pso_trace(self, f: torch.Tensor | None, pos: torch.Tensor | None = None,
                  gbest: torch.Tensor | None = None):
        """pifcm_pso_trace: f [G,P] f64, pos [G,P,2] f64, gbest [G] int32 (device),
        filled per generation by every later PSO update; None switches it off."""
        G = 0 if f is None else f.shape[0]
        self._ck(self.lib.pifcm_pso_trace(self._h, _ptr(f), _ptr(pos), _ptr(gbest), G))

    def pso_step(self, grid, cfg, pso, x, ws, stream=None):
        self._ck(self.lib.pifcm_pso_step(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                         _ptr(x), _ptr(ws), ws.numel(), _stream(stream)))

    def pso_fitness(self, grid, cfg, pso, ws) -> torch.Tensor:
        """The fp64 [P] fitness vector inside ws, as a tensor view (for all-gather)."""
        p = ct.c_void_p()
        self._ck(self.lib.pifcm_pso_fitness_ptr(ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                                _ptr(ws), ct.byref(p)))
        off = p.value - ws.data_ptr()
        return ws[off: off + 8 * pso.P].view(torch.float64)

    def pso_result(self, grid, cfg, pso, ws, stream=None):
        r = _abi.PsoResult()
        stopped = ct.c_int32()
        self._ck(self.lib.pifcm_pso_result_get(self._h, ct.byref(grid), ct.byref(cfg.c()),
                                               ct.byref(pso.c()), _ptr(ws), ct.byref(r),
                                               ct.byref(stopped), _stream(stream)))
        return PsoSummary(r.lambda_, r.xi, r.J, r.generations, r.gbest_particle,
                          list(r.centers)[:cfg.C]), bool(stopped.value)

    def pso_gbest_state(self, grid, cfg, pso, ws, U_out, c_out, stream=None):
        self._ck(self.lib.pifcm_pso_gbest_state(self._h, ct.byref(grid), ct.byref(cfg.c()),
                                                ct.byref(pso.c()), _ptr(ws), _ptr(U_out), _ptr(c_out),
                                                _stream(stream)))

    def pso_run(self, x, U0, c0, cfg, pso, nx, ws=None, stream=None) -> PsoSummary:
        nz, ny, pitch = x.shape
        g = _grid(nx, ny, nz, pitch)
        if ws is None:
            ws = self.workspace(nx, ny, nz, cfg, pso)
        r = _abi.PsoResult()
        self._ck(self.lib.pifcm_pso_run(self._h, ct.byref(g), ct.byref(cfg.c()), ct.byref(pso.c()),
                                        _ptr(x), _ptr(U0), _ptr(c0), _ptr(ws), ws.numel(), ct.byref(r),
                                        _stream(stream)))
        return PsoSummary(r.lambda_, r.xi, r.J, r.generations, r.gbest_particle,
                          list(r.centers)[:cfg.C])

    # ------------------------------------------------------------ pipeline parts
    def normalize(self, vol: torch.Tensor, want_hist=True, stream=None, mm=None):
        """pifcm_normalize: device u8 / uint16 / float32 volume [nz, ny, nx] ->
        (x [nz, ny, pitch] f32, R15 histogram int64 [256] or None).
        mm (optional device int32 tensor of >= 64 elements) receives the raw
        {min, max} in its first two entries (pifcm_fcm_hist's range)."""
        nz, ny, nx = vol.shape
        g = _grid(nx, ny, nz)
        x = torch.empty((nz, ny, g.pitch), dtype=torch.float32, device=vol.device)
        hist = torch.empty(256, dtype=torch.int64, device=vol.device) if want_hist else None
        ws = torch.empty(256, dtype=torch.uint8, device=vol.device) if mm is None else mm
        if ws.numel() * ws.element_size() < 256:
            raise ValueError("mm must hold >= 256 bytes")
        self._ck(self.lib.pifcm_normalize(self._h, ct.byref(g), _ptr(vol), dtype_code(vol), _ptr(x), _ptr(hist),
                                          _ptr(ws), 256, _stream(stream)))
        return x, hist

    # --------------------------------------- FCM start on the value histogram
    def value_hist(self, vol: torch.Tensor, counts: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """pifcm_value_hist: counts[v] += voxels of raw value v (uint8 -> 256,
        uint16 -> 65536 entries, int64).  A new zeroed tensor if counts is None."""
        code = dtype_code(vol)
        if counts is None:
            counts = torch.zeros(256 if code == _abi.U8 else 65536, dtype=torch.int64, device=vol.device)
        self._ck(self.lib.pifcm_value_hist(self._h, _ptr(vol), code, vol.numel(), _ptr(counts), _stream(stream)))
        return counts

    def fcm_hist(self, counts: torch.Tensor, mm: torch.Tensor, c0: torch.Tensor, cfg: IfcmConfig, stream=None):
        """pifcm_fcm_hist -> (c_prev [4], c_out [4], stats [4] = {J, du, iters, converged}),
        all device tensors."""
        code = _abi.U8 if counts.numel() == 256 else _abi.U16
        n = ct.c_size_t()
        self._ck(self.lib.pifcm_fcm_hist_workspace_size(code, ct.byref(n)))
        ws = torch.empty(n.value, dtype=torch.uint8, device=counts.device)
        c_prev = torch.zeros(4, dtype=torch.float32, device=counts.device)
        c_out = torch.zeros(4, dtype=torch.float32, device=counts.device)
        stats = torch.zeros(4, dtype=torch.float64, device=counts.device)
        self._ck(self.lib.pifcm_fcm_hist(self._h, ct.byref(cfg.c()), code, _ptr(mm), _ptr(counts), _ptr(c0),
                                         _ptr(c_prev), _ptr(c_out), _ptr(stats), _ptr(ws), n.value,
                                         _stream(stream)))
        return c_prev, c_out, stats

    def fcm_memberships(self, x: torch.Tensor, c: torch.Tensor, C: int, m: float, nx: int,
                        U: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """pifcm_fcm_memberships: U [nz*ny*nx, 4] = Eq. 2 rows of x (pitched
        [nz, ny, pitch]) at the centres c with lambda = xi = 0."""
        nz, ny, pitch = x.shape
        if U is None:
            U = torch.empty((nz * ny * nx, 4), dtype=torch.float32, device=x.device)
        g = _grid(nx, ny, nz, pitch)
        self._ck(self.lib.pifcm_fcm_memberships(self._h, ct.byref(g), C, m, _ptr(x), _ptr(c), _ptr(U),
                                                _stream(stream)))
        return U

    def normalize_u8(self, vol: torch.Tensor, want_hist=True, stream=None):
        if vol.dtype != torch.uint8:
            raise TypeError("normalize_u8 takes a uint8 volume (see normalize)")
        return self.normalize(vol, want_hist, stream)

    def gmm_init(self, hist: torch.Tensor, C: int, stream=None) -> torch.Tensor:
        c0 = torch.zeros(4, dtype=torch.float32, device=hist.device)
        self._ck(self.lib.pifcm_gmm_init(self._h, C, _ptr(hist), _ptr(c0), None, 0, _stream(stream)))
        return c0

    def incs(self, labels: torch.Tensor, truth: torch.Tensor, centers: torch.Tensor, C: int, stream=None) -> int:
        """pifcm_incs (R26): voxels whose label, mapped to a class by its
        centre's rank, differs from the phantom truth."""
        cnt = torch.zeros(1, dtype=torch.int64, device=labels.device)
        c = torch.zeros(4, dtype=torch.float32, device=labels.device)
        c[:C] = centers.reshape(-1)[:C].to(labels.device, torch.float32)
        self._ck(self.lib.pifcm_incs(self._h, _ptr(labels.contiguous()), _ptr(truth.contiguous()), labels.numel(),
                                     C, _ptr(c), _ptr(cnt), _stream(stream)))
        return int(cnt.item())

    def argmax(self, U: torch.Tensor, nx, ny, nz, C, stream=None) -> torch.Tensor:
        labels = torch.empty((nz, ny, nx), dtype=torch.uint8, device=U.device)
        g = _grid(nx, ny, nz)
        self._ck(self.lib.pifcm_argmax(self._h, ct.byref(g), C, _ptr(U), _ptr(labels), _stream(stream)))
        return labels

    # ------------------------------------------------------------ pipeline
    def segment(self, vol: torch.Tensor, cfg: IfcmConfig, pso: PsoConfig, ws=None, want_U=False,
                z_slice: int = -1, stream=None):
        """pifcm_segment on a device u8 / uint16 / float32 volume [nz, ny, nx]
        -> (labels, U or None, report)."""
        nz, ny, nx = vol.shape
        if ws is None:
            ws = self.workspace(nx, ny, nz, cfg, pso)
        if z_slice < 0:
            labels = torch.empty((nz, ny, nx), dtype=torch.uint8, device=vol.device)
        else:
            labels = torch.empty((ny, nx), dtype=torch.uint8, device=vol.device)
        U = torch.empty((nz * ny * nx, 4), dtype=torch.float32, device=vol.device) if want_U else None
        rep = _abi.Report()
        self._ck(self.lib.pifcm_segment(self._h, _ptr(vol), dtype_code(vol), nx, ny, nz, ct.byref(cfg.c()),
                                        ct.byref(pso.c()), z_slice, _ptr(ws), ws.numel(), _ptr(labels),
                                        _ptr(U), ct.byref(rep), _stream(stream)))
        return labels, U, report_dict(rep, cfg.C)

    def segment_slice(self, vol: torch.Tensor, z: int, cfg: IfcmConfig, pso: PsoConfig, want_U=False,
                      stream=None):
        """pifcm_segment_slice (literal slice mode, R25): slice z of a device
        uint8 volume [nz, ny, nx] with its 3D neighbourhood -> (labels [ny, nx],
        U [ny*nx, 4] or None, report)."""
        if vol.dtype != torch.uint8:
            raise TypeError("the slice mode takes uint8 volumes")
        nz, ny, nx = vol.shape
        n = ct.c_size_t()
        self._ck(self.lib.pifcm_segment_slice_workspace_size(nx, ny, nz, z, ct.byref(cfg.c()), ct.byref(pso.c()),
                                                             ct.byref(n)))
        ws = torch.empty(n.value, dtype=torch.uint8, device=vol.device)
        labels = torch.empty((ny, nx), dtype=torch.uint8, device=vol.device)
        U = torch.empty((ny * nx, 4), dtype=torch.float32, device=vol.device) if want_U else None
        rep = _abi.Report()
        self._ck(self.lib.pifcm_segment_slice(self._h, _ptr(vol.contiguous()), nx, ny, nz, z, ct.byref(cfg.c()),
                                              ct.byref(pso.c()), _ptr(ws), n.value, _ptr(labels), _ptr(U),
                                              ct.byref(rep), _stream(stream)))
        return labels, U, report_dict(rep, cfg.C)

    def segment_host(self, vol_host: torch.Tensor, cfg: IfcmConfig, pso: PsoConfig, ws,
                     labels_host: torch.Tensor, stream=None):
        """pifcm_segment_host: host (pinned) u8 volume in, host u8 labels out."""
        nz, ny, nx = vol_host.shape
        rep = _abi.Report()
        self._ck(self.lib.pifcm_segment_host(self._h, _ptr(vol_host), nx, ny, nz, ct.byref(cfg.c()),
                                             ct.byref(pso.c()), _ptr(ws), ws.numel(), _ptr(labels_host),
                                             ct.byref(rep), _stream(stream)))
        return report_dict(rep, cfg.C)


    # ------------------------------------------------------------ z-slab
    def slab_chunk(self, nx, ny, nz_total) -> int:
        """Planes per global z-chunk of the slab / canonical decomposition."""
        return slab_chunk(nx, ny, nz_total, self.lib)

    def slab_records(self, grid) -> int:
        n = ct.c_int32()
        self._ck(self.lib.pifcm_slab_records(ct.byref(grid), ct.byref(n)))
        return n.value

    def slab_step(self, grid, cfg, x, U_in, U_out, centers, lam_xi, records, stats=None, stream=None):
        P = U_in.shape[0]
        self._ck(self.lib.pifcm_slab_step(self._h, ct.byref(grid), ct.byref(cfg.c()), _ptr(x), _ptr(U_in),
                                          _ptr(U_out), _ptr(centers), _ptr(lam_xi), P, _ptr(stats),
                                          _ptr(records), _stream(stream)))

    def slab_finalize(self, C, P, world, nrec, records, centers, stats=None, fitness=None, eps=0.0,
                      counts=None, stream=None):
        """counts: device int32 [world] real records per rank (None: all nrec)."""
        self._ck(self.lib.pifcm_slab_finalize(self._h, C, P, world, nrec, _ptr(counts), _ptr(records),
                                              _ptr(centers), _ptr(stats), _ptr(fitness), eps, _stream(stream)))

    def slab_halo(self, grid, P, op, U, buf=None, stream=None, v=1):
        """pifcm_slab_halo_v: the v halo planes per side of P slab states."""
        self._ck(self.lib.pifcm_slab_halo_v(self._h, ct.byref(grid), v, P, op, _ptr(U), _ptr(buf),
                                            _stream(stream)))

    # ------------------------------------------------------- peer memory
    def peer_alloc(self, nbytes: int) -> int:
        """Zeroed device memory shareable with other processes (raw pointer)."""
        p = ct.c_void_p()
        self._ck(self.lib.pifcm_peer_alloc(self._h, nbytes, ct.byref(p)))
        return p.value

    def peer_free(self, ptr: int):
        self._ck(self.lib.pifcm_peer_free(self._h, ptr))

    def peer_handle(self, ptr: int) -> bytes:
        h = (ct.c_uint8 * 64)()
        self._ck(self.lib.pifcm_peer_handle(self._h, ptr, h))
        return bytes(h)

    def peer_open(self, handle: bytes) -> int:
        h = (ct.c_uint8 * 64).from_buffer_copy(handle)
        p = ct.c_void_p()
        self._ck(self.lib.pifcm_peer_open(self._h, h, ct.byref(p)))
        return p.value

    def peer_close(self, ptr: int):
        self._ck(self.lib.pifcm_peer_close(self._h, ptr))

    def slab_p2p_run(self, grid, cfg, x, peers, P, counts, nrec_max, centers, lam_xi, stats, rec_local, iters,
                     epoch: int, cur: int, stream=None):
        """pifcm_slab_p2p_run -> (epoch, cur, iters_done)."""
        e = ct.c_uint32(epoch)
        c = ct.c_int32(cur)
        n = ct.c_int32(0)
        self._ck(self.lib.pifcm_slab_p2p_run(self._h, ct.byref(grid), ct.byref(cfg.c()), _ptr(x), ct.byref(peers), P,
                                             _ptr(counts), nrec_max, _ptr(centers), _ptr(lam_xi), _ptr(stats),
                                             _ptr(rec_local), iters, ct.byref(e), ct.byref(c), ct.byref(n),
                                             _stream(stream)))
        return e.value, c.value, n.value

    # -------------------------------------------- pipeline parts for slab ranks
    def minmax_u8(self, vol: torch.Tensor, mm: torch.Tensor, stream=None):
        """mm: device int32 [2] <- {min, max} of vol (uint32 bits; values <= 255)."""
        self._ck(self.lib.pifcm_minmax_u8(self._h, _ptr(vol), vol.numel(), _ptr(mm), _stream(stream)))

    def normalize_u8_range(self, vol: torch.Tensor, mm: torch.Tensor, stream=None) -> torch.Tensor:
        nz, ny, nx = vol.shape
        g = _grid(nx, ny, nz)
        x = torch.zeros((nz, ny, g.pitch), dtype=torch.float32, device=vol.device)
        self._ck(self.lib.pifcm_normalize_u8_range(self._h, ct.byref(g), _ptr(vol), _ptr(mm), _ptr(x),
                                                   _stream(stream)))
        return x

    def hist_u8(self, vol: torch.Tensor, mm: torch.Tensor, stream=None) -> torch.Tensor:
        hist = torch.empty(256, dtype=torch.int64, device=vol.device)
        self._ck(self.lib.pifcm_hist_u8(self._h, _ptr(vol), vol.numel(), _ptr(mm), _ptr(hist), _stream(stream)))
        return hist

    # ------------------------------------------------- PSO over z-slab ranks
    def slab_workspace(self, grid, cfg, pso) -> torch.Tensor:
        n = ct.c_size_t()
        self._ck(self.lib.pifcm_slab_workspace_size(ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                                    ct.byref(n)))
        return torch.empty(n.value, dtype=torch.uint8, device=f"cuda:{self.device}")

    def slab_pso_init(self, grid, cfg, pso, U0, c0, ws, stream=None):
        self._ck(self.lib.pifcm_slab_pso_init(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                              _ptr(U0), _ptr(c0), _ptr(ws), ws.numel(), _stream(stream)))

    def slab_pso_halo(self, grid, cfg, pso, ws, op, buf=None, stream=None):
        self._ck(self.lib.pifcm_slab_pso_halo(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                              _ptr(ws), ws.numel(), op, _ptr(buf), _stream(stream)))

    def slab_pso_eval(self, grid, cfg, pso, x, ws, records, stream=None):
        self._ck(self.lib.pifcm_slab_pso_eval(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                              _ptr(x), _ptr(ws), ws.numel(), _ptr(records), _stream(stream)))

    def slab_pso_finalize(self, grid, cfg, pso, ws, world, nrec, records, counts=None, stream=None):
        self._ck(self.lib.pifcm_slab_pso_finalize(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                                  _ptr(ws), ws.numel(), world, nrec, _ptr(counts),
                                                  _ptr(records), _stream(stream)))

    def slab_pso_update(self, grid, cfg, pso, ws, stream=None):
        self._ck(self.lib.pifcm_slab_pso_update(self._h, ct.byref(grid), ct.byref(cfg.c()), ct.byref(pso.c()),
                                                _ptr(ws), ws.numel(), _stream(stream)))

    def slab_pso_result(self, grid, cfg, pso, ws, stream=None):
        r = _abi.PsoResult()
        stopped = ct.c_int32()
        self._ck(self.lib.pifcm_slab_pso_result_get(self._h, ct.byref(grid), ct.byref(cfg.c()),
                                                    ct.byref(pso.c()), _ptr(ws), ct.byref(r),
                                                    ct.byref(stopped), _stream(stream)))
        return PsoSummary(r.lambda_, r.xi, r.J, r.generations, r.gbest_particle,
                          list(r.centers)[:cfg.C]), bool(stopped.value)

    def slab_pso_gbest_state(self, grid, cfg, pso, ws, U_out, c_out, stream=None):
        self._ck(self.lib.pifcm_slab_pso_gbest_state(self._h, ct.byref(grid), ct.byref(cfg.c()),
                                                     ct.byref(pso.c()), _ptr(ws), _ptr(U_out), _ptr(c_out),
                                                     _stream(stream)))

    def slab_pso_fitness(self, grid, cfg, pso, ws) -> torch.Tensor:
        """Fitness vector of the slab swarm (a view into ws)."""
        pg = _grid(grid.nx, grid.ny, grid.nz + 2 * cfg.v, grid.pitch)  # the slab arrays: v halo planes per side
        return self.pso_fitness(pg, cfg, pso, ws)


def slab_chunk(nx, ny, nz_total, lib=None) -> int:
    """pifcm_slab_chunk (host-only query, no GPU needed)."""
    lib = lib or _abi.load()
    tz = ct.c_int32()
    rc = lib.pifcm_slab_chunk(nx, ny, nz_total, ct.byref(tz))
    if rc != 0:
        raise PifcmError(rc, "pifcm_slab_chunk: invalid dimensions")
    return tz.value


def eq11(incs_tab, secs_tab, alpha: float, lib=None) -> list:
    """pifcm_eq11: the Eq. 11 cost of each algorithm from [k sizes][A algorithms]
    tables of incS and seconds (host arithmetic in libpifcm.so)."""
    lib = lib or _abi.load()
    k, A = len(incs_tab), len(incs_tab[0])
    q = (ct.c_double * (k * A))(*[float(v) for row in incs_tab for v in row])
    t = (ct.c_double * (k * A))(*[float(v) for row in secs_tab for v in row])
    J = (ct.c_double * A)()
    rc = lib.pifcm_eq11(q, t, k, A, float(alpha), J)
    if rc != 0:
        raise PifcmError(rc, "pifcm_eq11: invalid tables or alpha")
    return list(J)


def report_dict(rep: _abi.Report, C: int) -> dict:
    return {
        "lambda": rep.pso.lambda_, "xi": rep.pso.xi, "J": rep.pso.J,
        "generations": rep.pso.generations, "gbest_particle": rep.pso.gbest_particle,
        "fcm_iters": rep.fcm_iters, "final_iters": rep.final_iters,
        "c_init": list(rep.c_init)[:C], "centers": list(rep.centers)[:C],
        "t_norm": rep.t_norm, "t_init": rep.t_init, "t_pso": rep.t_pso, "t_final": rep.t_final,
        "t_total": rep.t_total,
    }
