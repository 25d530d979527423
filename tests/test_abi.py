"""The C-ABI library loads and exports every symbol include/pifcm.h declares
(no compute calls: CPU only)."""
import ctypes as ct
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pifcm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pifcm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2002_01981_b200 import build
    build.build()
    return ct.CDLL(build.LIB)


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("pifcm_iterate", "pifcm_segment", "pifcm_pso_step", "pifcm_pso_run"):
        assert name in d


def test_exports_every_declared_symbol(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2002_01981_b200 import _abi
    assert sorted(_abi.SIGNATURES) == _declared()


def test_version_and_validation_without_gpu(lib):
    from paper_2002_01981_b200 import _abi
    L = _abi.load()
    assert b"sm_100a" in L.pifcm_version()
    g = _abi.Grid(181, 217, 181, 184, 0, 0)
    cfg = _abi.IfcmCfg(4, 2.0, 1, 1.0, 0, 1e-5, 100)
    pso = _abi.PsoCfg(32, 1, 30, 0, 1e-4, 0.1, 0.5, 1, 0, 0, 0)
    n = ct.c_size_t()
    assert L.pifcm_workspace_size(ct.byref(g), ct.byref(cfg), ct.byref(pso), ct.byref(n)) == 0
    nvox = 181 * 217 * 181
    assert n.value >= 16 * nvox * 65  # 2P+1 slots of AoS-C4 states
    bad = _abi.IfcmCfg(5, 2.0, 1, 1.0, 0, 1e-5, 100)
    assert L.pifcm_workspace_size(ct.byref(g), ct.byref(bad), None, ct.byref(n)) == -1
    badg = _abi.Grid(181, 217, 181, 181, 0, 0)
    assert L.pifcm_workspace_size(ct.byref(badg), ct.byref(cfg), None, ct.byref(n)) == -2
    badm = _abi.IfcmCfg(4, 1.0, 1, 1.0, 0, 1e-5, 100)
    assert L.pifcm_workspace_size(ct.byref(g), ct.byref(badm), None, ct.byref(n)) == -1


def test_struct_sizes_match_c():
    from paper_2002_01981_b200 import _abi
    assert ct.sizeof(_abi.Grid) == 24
    assert ct.sizeof(_abi.IfcmCfg) == 28
    assert ct.sizeof(_abi.PsoCfg) == 64
    assert ct.sizeof(_abi.PsoResult) == 48


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2002_01981_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "pifcm_oracle" not in txt and "liboracle" not in txt, f


def test_eq11_host_matches_oracle(orc):
    """pifcm_eq11 is host arithmetic in libpifcm.so (no GPU): equal to the
    oracle's Eq. 11 on random tables and on the hand-worked example."""
    import numpy as np
    from paper_2002_01981_b200.api import PifcmError, eq11
    g = np.random.default_rng(4)
    q = g.integers(0, 1000, size=(7, 5)).astype(float)
    t = g.random((7, 5)) * 100
    q[3] = 42.0  # a constant row
    for alpha in (0.0, 0.7, 1.0):
        assert np.allclose(eq11(q.tolist(), t.tolist(), alpha), orc.eq11(q, t, alpha), rtol=0, atol=1e-15)
    J = eq11([[10.0, 30.0, 20.0], [5.0, 5.0, 5.0]], [[1.0, 3.0, 2.0], [4.0, 2.0, 3.0]], 0.7)
    assert np.allclose(J, [0.15, 0.5, 0.325], rtol=0, atol=1e-15)
    import pytest
    with pytest.raises(PifcmError):
        eq11([[1.0]], [[1.0]], 1.5)


def test_dist_range_matches_shard_range():
    """pifcm_dist_range (C) is the split the Python drivers use (dist.shard_range)."""
    import ctypes as ct
    from paper_2002_01981_b200 import _abi
    from paper_2002_01981_b200.dist import shard_range
    lib = _abi.load()
    a, b = ct.c_int32(), ct.c_int32()
    for P in (1, 5, 20, 32, 33, 64):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert lib.pifcm_dist_range(P, world, r, ct.byref(a), ct.byref(b)) == 0
                assert (a.value, b.value) == shard_range(P, world, r)
    assert lib.pifcm_dist_range(4, 2, 2, ct.byref(a), ct.byref(b)) != 0
