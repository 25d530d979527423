"""The FCM start on the value histogram (DESIGN R24) against
the oracle's per-voxel FCM (oracle fcm_run: Alg. 1 step 2 / Alg. 2 step 5 at
lambda = xi = 0, every voxel, fp64), through the C ABI."""
import numpy as np
import pytest
import torch

from inputs import add_noise_u8, brainweb_phantom, cube_phantom

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def ctx():
    from paper_2002_01981_b200 import Context
    return Context(0)


def _fcm_gpu(ctx, vol, c0, C, m=2.0, eps=1e-5, max_iter=100):
    from paper_2002_01981_b200 import IfcmConfig
    cfg = IfcmConfig(C=C, m=m, eps=eps, max_iter=max_iter)
    vt = torch.as_tensor(vol, device=DEV)
    mm = torch.zeros(64, dtype=torch.int32, device=DEV)
    x, _ = ctx.normalize(vt, mm=mm)
    counts = ctx.value_hist(vt)
    c0t = torch.zeros(4, dtype=torch.float32, device=DEV)
    c0t[:C] = torch.as_tensor(np.asarray(c0, np.float32))
    c_prev, c_out, st = ctx.fcm_hist(counts, mm, c0t, cfg)
    nz, ny, nx = vol.shape
    U = ctx.fcm_memberships(x, c_prev, C, m, nx)
    return x[..., :nx].cpu().numpy(), U.cpu().numpy()[:, :C], c_out.cpu().numpy()[:C], st.cpu().numpy(), counts


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
@pytest.mark.parametrize("shape,seed", [((1, 9, 7), 1), ((6, 40, 33), 2), ((23, 31, 45), 3)])
def test_value_hist_bit_exact(ctx, dtype, shape, seed):
    g = np.random.default_rng(seed)
    hi = 256 if dtype == np.uint8 else 65536
    v = g.integers(0, hi, size=shape).astype(dtype)
    counts = ctx.value_hist(torch.as_tensor(v, device=DEV)).cpu().numpy()
    assert counts.shape[0] == hi
    assert (counts == np.bincount(v.ravel().astype(np.int64), minlength=hi)).all()
    # accumulates (the z-slab ranks' counts are summed the same way)
    t = torch.as_tensor(counts, device=DEV)
    ctx.value_hist(torch.as_tensor(v, device=DEV), t)
    assert (t.cpu().numpy() == 2 * counts).all()


@pytest.mark.parametrize("C,m,maker,seed", [
    (3, 2.0, lambda: cube_phantom(24, 20, 8, (0.1, 0.5, 0.9))[0], 1),
    (4, 2.0, lambda: cube_phantom(33, 29, 11)[0], 2),
    (4, 2.0, lambda: brainweb_phantom(45, 54, 45)[0], 3),
    (2, 2.0, lambda: cube_phantom(16, 16, 1, (0.2, 0.8))[0], 4),
    (4, 1.7, lambda: cube_phantom(30, 21, 7)[0], 5),
])
def test_fcm_hist_vs_oracle(ctx, orc, C, m, maker, seed):
    """Same x, same start centres: the GPU's iteration count, memberships
    (1e-4 abs, every voxel) and centres (1e-4 rel) against the oracle's
    per-voxel FCM with its eps stop; then against the oracle run for exactly
    the GPU's iteration count (the eps decision may flip on rounding)."""
    vol = add_noise_u8(maker(), 7.0, seed)
    c0 = np.linspace(0.15, 0.85, C)
    x, U, c, st, _ = _fcm_gpu(ctx, vol, c0, C, m=m)
    T = int(st[2])
    Uo, co, To = orc.fcm_run(x.astype(np.float64), c0.astype(np.float32).astype(np.float64), eps=1e-5, m=m)
    assert abs(T - To) <= 1, (T, To)
    assert st[3] == 1.0 and st[1] < 1e-5
    Uo, co, _ = orc.fcm_run(x.astype(np.float64), c0.astype(np.float32).astype(np.float64), eps=0.0,
                            max_iter=T, m=m)
    assert np.abs(U - Uo).max() < 1e-4
    assert np.allclose(c, co, rtol=1e-4, atol=0)
    assert np.allclose(U.sum(1), 1.0, atol=1e-6)


def test_fcm_hist_fixed_iterations_and_J(ctx, orc):
    """eps = 0: exactly max_iter iterations; J of the last iteration = the
    oracle's Eq. 1 cost of that step."""
    vol = add_noise_u8(cube_phantom(28, 22, 6)[0], 9.0, 7)
    c0 = np.array([0.1, 0.4, 0.6, 0.9])
    x, U, c, st, _ = _fcm_gpu(ctx, vol, c0, 4, eps=0.0, max_iter=5)
    assert int(st[2]) == 5 and st[3] == 0.0
    x64 = x.astype(np.float64).ravel()
    U4, c4, _ = orc.fcm_run(x64, c0.astype(np.float32).astype(np.float64), eps=0.0, max_iter=4)
    Un, cn, J, du = orc.fcm_step(x64, c4.astype(np.float32).astype(np.float64), U_old=U4)
    assert np.abs(U - Un).max() < 1e-4
    assert abs(st[0] - J) <= 1e-4 * J
    assert abs(st[1] - du) < 1e-4


def test_fcm_hist_constant_volume(ctx, orc):
    """R16: a constant volume normalises to x = 0 everywhere."""
    vol = np.full((3, 10, 12), 77, np.uint8)
    c0 = np.array([0.2, 0.5, 0.8])
    x, U, c, st, counts = _fcm_gpu(ctx, vol, c0, 3)
    assert (x == 0).all()
    assert int(counts[77].item()) == vol.size
    Uo, co, _ = orc.fcm_run(x.astype(np.float64), c0, eps=0.0, max_iter=int(st[2]))
    assert np.abs(U - Uo).max() < 1e-4
    assert np.allclose(c, co, rtol=1e-4, atol=1e-7)


def test_fcm_hist_u16_equals_u8(ctx):
    """v16 = 257 * v8 normalises to the same x, so the 65536-value histogram
    gives bit-identical centres, statistics and memberships."""
    v8 = add_noise_u8(cube_phantom(25, 19, 9)[0], 7.0, 11)
    c0 = np.array([0.1, 0.35, 0.65, 0.9])
    a = _fcm_gpu(ctx, v8, c0, 4)
    b = _fcm_gpu(ctx, v8.astype(np.uint16) * 257, c0, 4)
    for p, q in zip(a[:4], b[:4]):
        assert (p == q).all()
