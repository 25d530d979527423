"""ctypes marshalling for oracle/pifcm_oracle.c -- TEST INFRASTRUCTURE ONLY.

Every function takes and returns numpy fp64 arrays in the oracle's layouts:
``x`` [nz, ny, nx], ``U`` [N, C] (N = nz*ny*nx, x fastest), ``c`` [C].
No arithmetic of the method happens here; see pifcm_oracle.c for the
paper citations of each step.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pifcm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

__all__ = [
    "shell_weights", "ifcm_step", "ifcm_voxels", "fcm_step", "centers", "argmax",
    "normalize_u8", "histogram_u8", "normalize", "histogram", "gmm_init", "philox4x32_10", "philox_pair",
    "pso_init", "pso_move", "pso_update", "pso_run", "ifcm_run", "fcm_run", "segment_u8",
    "num_threads", "set_num_threads", "PsoResult", "SegmentResult",
    "ifcm_step_planes", "histogram_u8_range", "segment_slice_u8", "SliceResult", "incs", "eq11",
]


def lib_path() -> str:
    return _LIB


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = ct.CDLL(_LIB)
        _declare(_lib)
    return _lib


_dp = ct.POINTER(ct.c_double)
_i64p = ct.POINTER(ct.c_int64)
_u8p = ct.POINTER(ct.c_uint8)
_u32p = ct.POINTER(ct.c_uint32)
_ip = ct.POINTER(ct.c_int)


def _declare(L):
    i, d, l, u64 = ct.c_int, ct.c_double, ct.c_long, ct.c_uint64
    L.orc_shell_weights.argtypes = [i, d, _dp]
    L.orc_ifcm_step.argtypes = [_dp, i, i, i, i, d, d, d, i, i, d, _dp, _dp, _dp, _dp, _dp, _dp]
    L.orc_ifcm_voxels.argtypes = [_dp, i, i, i, i, d, d, d, i, i, d, _dp, _dp, _i64p, l,
                                  _dp, _dp, _dp, _dp]
    L.orc_fcm_step.argtypes = [_dp, l, i, d, _dp, _dp, _dp, _dp, _dp, _dp]
    L.orc_centers.argtypes = [_dp, l, i, d, _dp, _dp, _dp]
    L.orc_argmax.argtypes = [_dp, l, i, _u8p]
    L.orc_normalize_u8.argtypes = [_u8p, l, _dp]
    L.orc_histogram_u8.argtypes = [_u8p, l, _i64p]
    L.orc_normalize_u16.argtypes = [_vp, l, _dp]
    L.orc_histogram_u16.argtypes = [_vp, l, _i64p]
    L.orc_normalize_f32.argtypes = [_vp, l, _dp]
    L.orc_histogram_f32.argtypes = [_vp, l, _i64p]
    L.orc_segment_typed.argtypes = [_vp, i, i, i, i, i, d, i, i, d, d, i, i, i, i, i, d, d, d, u64,
                                    _u8p, _dp, _dp, _dp, _dp, _ip, _ip, _dp, i]
    L.orc_segment_typed.restype = i
    L.orc_gmm_init.argtypes = [_i64p, i, i, _dp]
    L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.orc_philox_pair.argtypes = [u64, ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.c_uint32, _dp, _dp]
    L.orc_pso_init.argtypes = [i, u64, d, _dp, _dp]
    L.orc_pso_move.argtypes = [i, d, _dp, _dp, _ip, _dp, _dp, _dp]
    L.orc_pso_update.argtypes = [i, i, ct.c_uint32, u64, d, _dp, _dp, _dp, _dp, _dp, _ip, _ip]
    L.orc_pso_run.argtypes = [_dp, i, i, i, i, d, i, i, d, _dp, _dp, i, i, i, i, d, d, d, u64,
                              _dp, _dp, _dp, _dp, _dp, _dp, _ip, i]
    L.orc_pso_run.restype = i
    L.orc_ifcm_run.argtypes = [_dp, i, i, i, i, d, d, d, i, i, d, d, i, _dp, _dp, _dp]
    L.orc_ifcm_run.restype = i
    L.orc_fcm_run.argtypes = [_dp, l, i, d, d, i, _dp, _dp, _dp]
    L.orc_fcm_run.restype = i
    L.orc_segment_u8.argtypes = [_u8p, i, i, i, i, d, i, i, d, d, i, i, i, i, i, d, d, d, u64,
                                 _u8p, _dp, _dp, _dp, _dp, _ip, _ip, _dp, i]
    L.orc_segment_u8.restype = i
    L.orc_ifcm_step_planes.argtypes = [_dp, i, i, i, i, i, i, d, d, d, i, i, d, _dp, _dp, _dp, _dp, _dp, _dp]
    L.orc_histogram_u8_range.argtypes = [_u8p, l, i, i, _i64p]
    L.orc_segment_slice_u8.argtypes = [_u8p, i, i, i, i, i, d, i, i, d, d, i, i, i, i, i, d, d, d, u64,
                                       _u8p, _dp, _dp, _dp, _dp, _ip, _ip, _dp, _ip]
    L.orc_segment_slice_u8.restype = i
    L.orc_incs.argtypes = [_u8p, _u8p, l, i, _dp]
    L.orc_incs.restype = l
    L.orc_eq11.argtypes = [_dp, _dp, i, i, d, _dp]
    L.orc_num_threads.restype = i
    L.orc_set_num_threads.argtypes = [i]


_vp = ct.c_void_p


def _p(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return _L().orc_num_threads()


def set_num_threads(n: int) -> None:
    _L().orc_set_num_threads(int(n))


def shell_weights(v: int, h: float) -> np.ndarray:
    W = np.zeros(v, np.float64)
    _L().orc_shell_weights(v, h, _p(W))
    return W


def ifcm_step(x, U, c, lam, xi, m=2.0, q_mode=0, v=1, h=1.0):
    """One IFCM step. x [nz,ny,nx]; U [N,C]; c [C] -> (U_new, c_new, J, maxdu)."""
    x = _f64(x)
    nz, ny, nx = x.shape
    U = _f64(U)
    C = U.shape[1]
    c = _f64(c)
    Un = np.empty_like(U)
    cn = np.empty(C, np.float64)
    J = ct.c_double()
    du = ct.c_double()
    _L().orc_ifcm_step(_p(x), nx, ny, nz, C, m, lam, xi, q_mode, v, h, _p(U), _p(c),
                       _p(Un), _p(cn), ct.byref(J), ct.byref(du))
    return Un, cn, J.value, du.value


def ifcm_step_planes(x, U, c, lam, xi, zt0, zt1, m=2.0, q_mode=0, v=1, h=1.0):
    """One IFCM step of the target planes [zt0, zt1) only (R25): the other rows
    are copied; c, J, maxdu over the target planes."""
    x = _f64(x)
    nz, ny, nx = x.shape
    U = _f64(U)
    C = U.shape[1]
    c = _f64(c)
    Un = np.empty_like(U)
    cn = np.empty(C, np.float64)
    J = ct.c_double()
    du = ct.c_double()
    _L().orc_ifcm_step_planes(_p(x), nx, ny, nz, zt0, zt1, C, m, lam, xi, q_mode, v, h, _p(U), _p(c),
                              _p(Un), _p(cn), ct.byref(J), ct.byref(du))
    return Un, cn, J.value, du.value


def histogram_u8_range(vol, lo, hi):
    vol = np.ascontiguousarray(vol, dtype=np.uint8).ravel()
    h = np.empty(256, np.int64)
    _L().orc_histogram_u8_range(_p(vol, _u8p), vol.size, int(lo), int(hi), _p(h, _i64p))
    return h


def ifcm_voxels(x, U, c, lam, xi, idx, m=2.0, q_mode=0, v=1, h=1.0):
    """Per-voxel evaluation at flat voxel indices idx -> (u, d2, H, F), each [n, C]."""
    x = _f64(x)
    nz, ny, nx = x.shape
    U = _f64(U)
    C = U.shape[1]
    c = _f64(c)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    n = idx.shape[0]
    out = [np.empty((n, C), np.float64) for _ in range(4)]
    _L().orc_ifcm_voxels(_p(x), nx, ny, nz, C, m, lam, xi, q_mode, v, h, _p(U), _p(c),
                         _p(idx, _i64p), n, *[_p(o) for o in out])
    return tuple(out)


def fcm_step(x, c, m=2.0, U_old=None):
    """Standard FCM step (independent code path) -> (U_new, c_new, J, maxdu)."""
    x = _f64(x).ravel()
    c = _f64(c)
    C = c.shape[0]
    N = x.shape[0]
    Un = np.empty((N, C), np.float64)
    cn = np.empty(C, np.float64)
    J = ct.c_double()
    du = ct.c_double()
    Uo = _f64(U_old) if U_old is not None else None
    _L().orc_fcm_step(_p(x), N, C, m, _p(c), _p(Uo), _p(Un), _p(cn), ct.byref(J), ct.byref(du))
    return Un, cn, J.value, du.value


def centers(x, U, c_old, m=2.0):
    x = _f64(x).ravel()
    U = _f64(U)
    C = U.shape[1]
    cn = np.empty(C, np.float64)
    _L().orc_centers(_p(x), x.shape[0], C, m, _p(U), _p(_f64(c_old)), _p(cn))
    return cn


def argmax(U):
    U = _f64(U)
    N, C = U.shape
    lab = np.empty(N, np.uint8)
    _L().orc_argmax(_p(U), N, C, _p(lab, _u8p))
    return lab


def normalize_u8(vol):
    vol = np.ascontiguousarray(vol, dtype=np.uint8)
    x = np.empty(vol.shape, np.float64)
    _L().orc_normalize_u8(_p(vol, _u8p), vol.size, _p(x))
    return x


def histogram_u8(vol):
    vol = np.ascontiguousarray(vol, dtype=np.uint8)
    h = np.zeros(256, np.int64)
    _L().orc_histogram_u8(_p(vol, _u8p), vol.size, _p(h, _i64p))
    return h


_TYPED = {np.dtype(np.uint8): (0, "u8"), np.dtype(np.uint16): (1, "u16"), np.dtype(np.float32): (2, "f32")}


def normalize(vol):
    """Alg. 2 step 1 for a u8 / u16 / f32 volume (R16)."""
    vol = np.ascontiguousarray(vol)
    code, name = _TYPED[vol.dtype]
    x = np.empty(vol.shape, np.float64)
    ptr = vol.ctypes.data_as(_u8p if code == 0 else _vp)
    getattr(_L(), "orc_normalize_" + name)(ptr, vol.size, _p(x))
    return x


def histogram(vol):
    """R15 histogram of a u8 / u16 / f32 volume."""
    vol = np.ascontiguousarray(vol)
    code, name = _TYPED[vol.dtype]
    h = np.zeros(256, np.int64)
    ptr = vol.ctypes.data_as(_u8p if code == 0 else _vp)
    getattr(_L(), "orc_histogram_" + name)(ptr, vol.size, _p(h, _i64p))
    return h


def gmm_init(hist, C, max_iter=100):
    hist = np.ascontiguousarray(hist, dtype=np.int64)
    c0 = np.empty(C, np.float64)
    _L().orc_gmm_init(_p(hist, _i64p), C, max_iter, _p(c0))
    return c0


def philox4x32_10(ctr, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32)
    key = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.empty(4, np.uint32)
    _L().orc_philox4x32_10(_p(ctr, _u32p), _p(key, _u32p), _p(out, _u32p))
    return out


def philox_pair(seed, c0, c1, c2, c3):
    a = ct.c_double()
    b = ct.c_double()
    _L().orc_philox_pair(seed, c0, c1, c2, c3, ct.byref(a), ct.byref(b))
    return a.value, b.value


def pso_init(P, seed, v0=0.1):
    pos = np.empty((P, 2), np.float64)
    vel = np.empty((P, 2), np.float64)
    _L().orc_pso_init(P, seed, v0, _p(pos), _p(vel))
    return pos, vel


def pso_move(pos, vel, pbest_x, lbest, p1, p2, vmax=0.5):
    """In-place Alg. 1 steps 7-8 with explicit draws (for pinning the formula)."""
    P = pos.shape[0]
    lb = np.ascontiguousarray(lbest, dtype=np.int32)
    _L().orc_pso_move(P, vmax, _p(_f64(p1)), _p(_f64(p2)), lb.ctypes.data_as(_ip),
                      _p(_f64(pbest_x)), _p(pos), _p(vel))


def pso_update(f, pos, vel, pbest_f, pbest_x, gbest, gen, seed, ring_k=1, vmax=0.5):
    """In-place PSO update; returns (gbest, improved)."""
    P = pos.shape[0]
    f = _f64(f)
    g = ct.c_int(gbest)
    imp = ct.c_int(0)
    _L().orc_pso_update(P, ring_k, gen, seed, vmax, _p(f), _p(pos), _p(vel), _p(pbest_f),
                        _p(pbest_x), ct.byref(g), ct.byref(imp))
    return g.value, imp.value


@dataclass
class PsoResult:
    lam: float
    xi: float
    J: float
    U: np.ndarray
    c: np.ndarray
    generations: int
    trace_pos: np.ndarray
    trace_f: np.ndarray
    trace_gbest: np.ndarray


def pso_run(x, U0, c0, P, max_gen, seed, m=2.0, q_mode=0, v=1, h=1.0, ring_k=1, patience=0,
            tol=1e-4, v0=0.1, vmax=0.5, fitness_mode=0):
    """fitness_mode: 0 CHAINED, 1 ANCHORED, 2 LEADER (pifcm_oracle.c orc_pso_run)."""
    x = _f64(x)
    nz, ny, nx = x.shape
    U0 = _f64(U0)
    C = U0.shape[1]
    c0 = _f64(c0)
    lx = np.zeros(2)
    J = ct.c_double()
    Ub = np.empty_like(U0)
    cb = np.empty(C)
    tp = np.zeros((max_gen, P, 2))
    tf = np.zeros((max_gen, P))
    tg = np.zeros(max_gen, np.int32)
    gens = _L().orc_pso_run(_p(x), nx, ny, nz, C, m, q_mode, v, h, _p(U0), _p(c0), P, ring_k,
                            max_gen, patience, tol, v0, vmax, seed, _p(lx), ct.byref(J), _p(Ub),
                            _p(cb), _p(tp), _p(tf), tg.ctypes.data_as(_ip), fitness_mode)
    return PsoResult(lx[0], lx[1], J.value, Ub, cb, gens, tp[:gens], tf[:gens], tg[:gens])


def ifcm_run(x, U, c, lam, xi, eps=1e-5, max_iter=100, m=2.0, q_mode=0, v=1, h=1.0):
    x = _f64(x)
    nz, ny, nx = x.shape
    U = _f64(U).copy()
    c = _f64(c).copy()
    J = ct.c_double()
    it = _L().orc_ifcm_run(_p(x), nx, ny, nz, U.shape[1], m, lam, xi, q_mode, v, h, eps,
                           max_iter, _p(U), _p(c), ct.byref(J))
    return U, c, it, J.value


def fcm_run(x, c0, eps=1e-5, max_iter=100, m=2.0):
    x = _f64(x).ravel()
    c0 = _f64(c0)
    C = c0.shape[0]
    U = np.empty((x.shape[0], C))
    c = np.empty(C)
    t = _L().orc_fcm_run(_p(x), x.shape[0], C, m, eps, max_iter, _p(c0), _p(U), _p(c))
    return U, c, t


@dataclass
class SegmentResult:
    labels: np.ndarray
    U: np.ndarray
    c: np.ndarray
    lam: float
    xi: float
    J: float
    generations: int
    final_iters: int
    c_init: np.ndarray


def segment_u8(vol, C, P, max_gen, seed, m=2.0, q_mode=0, v=1, h=1.0, eps=1e-5, max_iter=100,
               ring_k=1, patience=0, tol=1e-4, v0=0.1, vmax=0.5, want_U=True, fitness_mode=0):
    vol = np.ascontiguousarray(vol)
    if vol.dtype not in _TYPED:
        vol = vol.astype(np.uint8)
    nz, ny, nx = vol.shape
    N = vol.size
    lab = np.empty(N, np.uint8)
    U = np.empty((N, C)) if want_U else None
    c = np.empty(C)
    lx = np.empty(2)
    J = ct.c_double()
    gens = ct.c_int()
    fi = ct.c_int()
    ci = np.empty(C)
    code = _TYPED[vol.dtype][0]
    _L().orc_segment_typed(vol.ctypes.data_as(_vp), code, nx, ny, nz, C, m, q_mode, v, h, eps, max_iter, P,
                           ring_k, max_gen, patience, tol, v0, vmax, seed, _p(lab, _u8p), _p(U), _p(c),
                           _p(lx), ct.byref(J), ct.byref(gens), ct.byref(fi), _p(ci), fitness_mode)
    return SegmentResult(lab.reshape(nz, ny, nx), U, c, lx[0], lx[1], J.value, gens.value,
                         fi.value, ci)


@dataclass
class SliceResult:
    labels: np.ndarray   # [ny, nx]
    U: np.ndarray        # [ny*nx, C]
    c: np.ndarray
    lam: float
    xi: float
    J: float
    generations: int
    final_iters: int
    c_init: np.ndarray
    fcm_iters: int


def segment_slice_u8(vol, z, C, P, max_gen, seed, m=2.0, q_mode=0, eps=1e-5, max_iter=100, ring_k=1,
                     patience=0, tol=1e-4, v0=0.1, vmax=0.5, v=1, h=1.0):
    """The literal slice mode (R25, orc_segment_slice_u8): segment slice z of a
    u8 volume [nz, ny, nx] with its 3D neighbourhood of radius v (Eq. 9-10;
    the neighbour planes z - v .. z + v fixed at the FCM rows)."""
    vol = np.ascontiguousarray(vol, dtype=np.uint8)
    nz, ny, nx = vol.shape
    n = nx * ny
    lab = np.empty(n, np.uint8)
    U = np.empty((n, C))
    c = np.empty(C)
    lx = np.empty(2)
    J = ct.c_double()
    gens = ct.c_int()
    fi = ct.c_int()
    ci = np.empty(C)
    fc = ct.c_int()
    r = _L().orc_segment_slice_u8(_p(vol, _u8p), nx, ny, nz, int(z), C, m, q_mode, int(v), float(h), eps,
                                  max_iter, P, ring_k,
                                  max_gen, patience, tol, v0, vmax, seed, _p(lab, _u8p), _p(U), _p(c), _p(lx),
                                  ct.byref(J), ct.byref(gens), ct.byref(fi), _p(ci), ct.byref(fc))
    if r != 0:
        raise ValueError(f"slice {z} outside [0, {nz})")
    return SliceResult(lab.reshape(ny, nx), U, c, lx[0], lx[1], J.value, gens.value, fi.value, ci, fc.value)


def incs(labels, truth, centers):
    """incS (R26): voxels whose label, mapped to a class by its centre's rank, differs from truth."""
    lab = np.ascontiguousarray(labels, dtype=np.uint8).ravel()
    tru = np.ascontiguousarray(truth, dtype=np.uint8).ravel()
    c = _f64(centers)
    return int(_L().orc_incs(_p(lab, _u8p), _p(tru, _u8p), lab.size, c.shape[0], _p(c)))


def eq11(incs_tab, secs_tab, alpha):
    """Eq. 11 cost per algorithm from [k sizes][A algorithms] tables of incS and seconds."""
    q = _f64(incs_tab)
    t = _f64(secs_tab)
    k, A = q.shape
    J = np.empty(A)
    _L().orc_eq11(_p(q), _p(t), k, A, float(alpha), _p(J))
    return J
