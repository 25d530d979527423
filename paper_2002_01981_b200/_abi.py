"""ctypes declarations of libpifcm.so (include/pifcm.h).  Marshalling only.

Loading fails loudly (RuntimeError) when the library has not been built:
there is no fallback implementation of any kind.
"""
from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpifcm.so")

PIFCM_OK = 0
STATUS = {0: "PIFCM_OK", -1: "PIFCM_EINVAL", -2: "PIFCM_EALIGN", -3: "PIFCM_ENOMEM",
          -4: "PIFCM_ECUDA", -5: "PIFCM_ENCCL", -6: "PIFCM_ENUMERIC", -7: "PIFCM_ESTATE"}
Q_LITERAL, Q_SQEUCLID = 0, 1
FIT_CHAINED = 0
FIT_ANCHORED = 1
FIT_LEADER = 2
ITER_CANONICAL = 1  # pifcm_iterate_ex flags
ITER_PER_STEP = 2
U8 = 0
U16 = 1
F32 = 2


class Grid(ct.Structure):
    _fields_ = [("nx", ct.c_int32), ("ny", ct.c_int32), ("nz", ct.c_int32), ("pitch", ct.c_int32),
                ("z0", ct.c_int32), ("nz_total", ct.c_int32)]


class IfcmCfg(ct.Structure):
    _fields_ = [("C", ct.c_int32), ("m", ct.c_float), ("v", ct.c_int32), ("h", ct.c_float),
                ("q_mode", ct.c_int32), ("eps", ct.c_float), ("max_iter", ct.c_int32)]


class PsoCfg(ct.Structure):
    _fields_ = [("P", ct.c_int32), ("ring_k", ct.c_int32), ("max_gen", ct.c_int32),
                ("patience", ct.c_int32), ("tol", ct.c_double), ("v0", ct.c_double),
                ("vmax", ct.c_double), ("seed", ct.c_uint64), ("fitness_mode", ct.c_int32),
                ("p_begin", ct.c_int32), ("p_end", ct.c_int32), ("eval_batch", ct.c_int32)]


class PsoResult(ct.Structure):
    _fields_ = [("lambda_", ct.c_double), ("xi", ct.c_double), ("J", ct.c_double),
                ("generations", ct.c_int32), ("gbest_particle", ct.c_int32),
                ("centers", ct.c_float * 4)]


class Report(ct.Structure):
    _fields_ = [("pso", PsoResult), ("fcm_iters", ct.c_int32), ("final_iters", ct.c_int32),
                ("c_init", ct.c_float * 4), ("centers", ct.c_float * 4),
                ("t_norm", ct.c_double), ("t_init", ct.c_double), ("t_pso", ct.c_double),
                ("t_final", ct.c_double), ("t_total", ct.c_double)]


class Dist(ct.Structure):
    _fields_ = [("rank", ct.c_int32), ("world", ct.c_int32), ("nccl_unique_id", ct.c_void_p),
                ("shard", ct.c_int32)]


HOST_ALLGATHER = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_size_t)
HOST_BROADCAST = ct.CFUNCTYPE(ct.c_int, ct.c_void_p, ct.c_void_p, ct.c_size_t, ct.c_int32)


class HostColl(ct.Structure):
    _fields_ = [("user", ct.c_void_p), ("allgather", HOST_ALLGATHER), ("broadcast", HOST_BROADCAST)]


MAX_PEERS = 16


class Peers(ct.Structure):
    """pifcm_peers: every rank's buffers as mapped into this process."""
    _fields_ = [("world", ct.c_int32), ("rank", ct.c_int32),
                ("U", (ct.c_void_p * MAX_PEERS) * 2), ("rec", (ct.c_void_p * MAX_PEERS) * 2),
                ("flags", ct.c_void_p * MAX_PEERS), ("nz", ct.c_int32 * MAX_PEERS)]


_vp = ct.c_void_p
_G = ct.POINTER(Grid)
_C = ct.POINTER(IfcmCfg)
_P = ct.POINTER(PsoCfg)

# name -> (restype, argtypes); the complete list of symbols include/pifcm.h declares
SIGNATURES = {
    "pifcm_version": (ct.c_char_p, []),
    "pifcm_ctx_create": (ct.c_int, [ct.c_int, ct.POINTER(_vp)]),
    "pifcm_ctx_destroy": (None, [_vp]),
    "pifcm_last_error": (ct.c_char_p, [_vp]),
    "pifcm_launch_count": (ct.c_int64, [_vp]),
    "pifcm_timing_enable": (ct.c_int, [_vp, ct.c_int32]),
    "pifcm_timing_read": (ct.c_int, [_vp, ct.c_int32, ct.POINTER(ct.c_double), ct.POINTER(ct.c_int64),
                                     ct.POINTER(ct.c_double)]),
    "pifcm_workspace_size": (ct.c_int, [_G, _C, _P, ct.POINTER(ct.c_size_t)]),
    "pifcm_iterate_workspace_size": (ct.c_int, [_G, _C, ct.c_int32, ct.c_int32, ct.POINTER(ct.c_size_t)]),
    "pifcm_iterate": (ct.c_int, [_vp, _G, _C, _vp, _vp, _vp, _vp, _vp, ct.c_int32, ct.c_int32, _vp,
                                 _vp, ct.c_size_t, _vp]),
    "pifcm_iterate_ex": (ct.c_int, [_vp, _G, _C, _vp, _vp, _vp, _vp, _vp, ct.c_int32, ct.c_int32, _vp,
                                 _vp, ct.c_size_t, ct.c_int32, _vp]),
    "pifcm_pso_init": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_pso_eval": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_pso_fitness_ptr": (ct.c_int, [_G, _C, _P, _vp, ct.POINTER(_vp)]),
    "pifcm_pso_update": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_pso_trace": (ct.c_int, [_vp, _vp, _vp, _vp, ct.c_int32]),
    "pifcm_nccl_unique_id": (ct.c_int, [_vp]),
    "pifcm_ctx_dist": (ct.c_int, [_vp, ct.POINTER(Dist), ct.POINTER(HostColl)]),
    "pifcm_dist_range": (ct.c_int, [ct.c_int32, ct.c_int32, ct.c_int32, ct.POINTER(ct.c_int32),
                                    ct.POINTER(ct.c_int32)]),
    "pifcm_pso_step": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_pso_result_get": (ct.c_int, [_vp, _G, _C, _P, _vp, ct.POINTER(PsoResult),
                                        ct.POINTER(ct.c_int32), _vp]),
    "pifcm_pso_gbest_state": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, _vp, _vp]),
    "pifcm_pso_run": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, _vp, _vp, ct.c_size_t,
                                 ct.POINTER(PsoResult), _vp]),
    "pifcm_normalize": (ct.c_int, [_vp, _G, _vp, ct.c_int32, _vp, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_normalize_u8": (ct.c_int, [_vp, _G, _vp, _vp, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_gmm_init": (ct.c_int, [_vp, ct.c_int32, _vp, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_argmax": (ct.c_int, [_vp, _G, ct.c_int32, _vp, _vp, _vp]),
    "pifcm_incs": (ct.c_int, [_vp, _vp, _vp, ct.c_int64, ct.c_int32, _vp, _vp, _vp]),
    "pifcm_eq11": (ct.c_int, [ct.POINTER(ct.c_double), ct.POINTER(ct.c_double), ct.c_int32, ct.c_int32,
                              ct.c_double, ct.POINTER(ct.c_double)]),
    "pifcm_value_hist": (ct.c_int, [_vp, _vp, ct.c_int32, ct.c_int64, _vp, _vp]),
    "pifcm_fcm_hist_workspace_size": (ct.c_int, [ct.c_int32, ct.POINTER(ct.c_size_t)]),
    "pifcm_fcm_hist": (ct.c_int, [_vp, _C, ct.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_fcm_memberships": (ct.c_int, [_vp, _G, ct.c_int32, ct.c_float, _vp, _vp, _vp, _vp]),
    "pifcm_segment": (ct.c_int, [_vp, _vp, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, _C, _P,
                                 ct.c_int32, _vp, ct.c_size_t, _vp, _vp, ct.POINTER(Report), _vp]),
    "pifcm_segment_host": (ct.c_int, [_vp, _vp, ct.c_int32, ct.c_int32, ct.c_int32, _C, _P, _vp,
                                      ct.c_size_t, _vp, ct.POINTER(Report), _vp]),
    "pifcm_segment_slice_workspace_size": (ct.c_int, [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, _C, _P,
                                                       ct.POINTER(ct.c_size_t)]),
    "pifcm_segment_slice": (ct.c_int, [_vp, _vp, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, _C, _P, _vp,
                                       ct.c_size_t, _vp, _vp, ct.POINTER(Report), _vp]),
    "pifcm_minmax_u8": (ct.c_int, [_vp, _vp, ct.c_int64, _vp, _vp]),
    "pifcm_normalize_u8_range": (ct.c_int, [_vp, _G, _vp, _vp, _vp, _vp]),
    "pifcm_hist_u8": (ct.c_int, [_vp, _vp, ct.c_int64, _vp, _vp, _vp]),
    "pifcm_slab_workspace_size": (ct.c_int, [_G, _C, _P, _vp]),
    "pifcm_slab_pso_init": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, _vp, ct.c_size_t, _vp]),
    "pifcm_slab_pso_halo": (ct.c_int, [_vp, _G, _C, _P, _vp, ct.c_size_t, ct.c_int32, _vp, _vp]),
    "pifcm_slab_pso_eval": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, ct.c_size_t, _vp, _vp]),
    "pifcm_slab_pso_finalize": (ct.c_int, [_vp, _G, _C, _P, _vp, ct.c_size_t, ct.c_int32, ct.c_int32, _vp, _vp,
                                           _vp]),
    "pifcm_slab_pso_update": (ct.c_int, [_vp, _G, _C, _P, _vp, ct.c_size_t, _vp]),
    "pifcm_slab_pso_result_get": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, _vp, _vp]),
    "pifcm_slab_pso_gbest_state": (ct.c_int, [_vp, _G, _C, _P, _vp, _vp, _vp, _vp]),
    "pifcm_peer_alloc": (ct.c_int, [_vp, ct.c_size_t, ct.POINTER(ct.c_void_p)]),
    "pifcm_peer_free": (ct.c_int, [_vp, _vp]),
    "pifcm_peer_handle": (ct.c_int, [_vp, _vp, _vp]),
    "pifcm_peer_open": (ct.c_int, [_vp, _vp, ct.POINTER(ct.c_void_p)]),
    "pifcm_peer_close": (ct.c_int, [_vp, _vp]),
    "pifcm_slab_p2p_run": (ct.c_int, [_vp, _G, _C, _vp, ct.POINTER(Peers), ct.c_int32, _vp, ct.c_int32, _vp, _vp,
                                      _vp, _vp, ct.c_int32, ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_int32),
                                      ct.POINTER(ct.c_int32), _vp]),
    "pifcm_slab_chunk": (ct.c_int, [ct.c_int32, ct.c_int32, ct.c_int32, _vp]),
    "pifcm_slab_records": (ct.c_int, [_G, ct.POINTER(ct.c_int32)]),
    "pifcm_slab_step": (ct.c_int, [_vp, _G, _C, _vp, _vp, _vp, _vp, _vp, ct.c_int32, _vp, _vp, _vp]),
    "pifcm_slab_finalize": (ct.c_int, [_vp, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, _vp, _vp, _vp,
                                       _vp, _vp, ct.c_float, _vp]),
    "pifcm_slab_halo": (ct.c_int, [_vp, _G, ct.c_int32, ct.c_int32, _vp, _vp, _vp]),
    "pifcm_slab_halo_v": (ct.c_int, [_vp, _G, ct.c_int32, ct.c_int32, ct.c_int32, _vp, _vp, _vp]),
}

_lib = None


def load(path: str | None = None) -> ct.CDLL:
    """Load libpifcm.so; raise if it is missing (no fallback exists).
    PIFCM_LIB may name a tuning variant built by build.py --out=..."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("PIFCM_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(
            f"libpifcm.so not found at {path}: build it with `python -m paper_2002_01981_b200.build` "
            "(there is no CPU or PyTorch fallback)")
    lib = ct.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
