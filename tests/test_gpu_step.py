"""GPU parity of the fused IFCM step (pifcm_iterate, through the C ABI) against
the fp64 oracle, from the same state (north_star tolerances: memberships 1e-4
absolute, centres 1e-4 relative).  The oracle receives the GPU's fp32 inputs
widened exactly to fp64."""
import numpy as np
import pytest
import torch

from inputs import random_state

pytestmark = pytest.mark.gpu

U_TOL = 1e-4
C_TOL = 1e-4


@pytest.fixture(scope="module")
def ctx():
    from paper_2002_01981_b200 import Context
    return Context(0)


def gpu_step(ctx, x, Us, cs, lamxi, C, m=2.0, q_mode=0, iters=1, eps=0.0, v=1, h=1.0):
    """Run `iters` iterations for P states; returns (U_new [P,N,C] f64, c [P,C], stats [P,4])."""
    from paper_2002_01981_b200 import IfcmConfig, to_aos, to_pitched_x
    dev = torch.device("cuda:0")
    nz, ny, nx = x.shape
    P = len(Us)
    xt = to_pitched_x(x, dev)
    Uin = to_aos(np.stack(Us), dev)
    Uout = torch.full_like(Uin, float("nan"))
    cen = torch.zeros((P, 4), dtype=torch.float32, device=dev)
    cen[:, :C] = torch.as_tensor(np.stack(cs), dtype=torch.float32)
    lx = torch.as_tensor(np.asarray(lamxi, np.float64).reshape(P, 2), device=dev)
    stats = torch.zeros((P, 4), dtype=torch.float64, device=dev)
    cfg = IfcmConfig(C=C, m=m, q_mode=q_mode, eps=eps, v=v, h=h)
    ctx.iterate(xt, Uin, Uout, cen, lx, cfg, iters=iters, stats=stats, nx=nx)
    torch.cuda.synchronize()
    U = Uout.cpu().numpy().astype(np.float64)
    assert np.isfinite(U).all()
    assert (U[..., C:] == 0).all()
    return U[..., :C], cen[:, :C].cpu().numpy().astype(np.float64), stats.cpu().numpy()


CASES = [
    # (nz, ny, nx), C, m, q_mode
    ((1, 8, 8), 2, 2.0, 0),
    ((5, 12, 12), 3, 2.0, 0),
    ((9, 17, 33), 4, 2.0, 0),
    ((19, 37, 70), 4, 2.0, 1),      # several tiles in x, y and z with ragged tails
    ((17, 16, 32), 3, 1.5, 0),      # exact tile multiples, z chunk + 1
    ((3, 50, 7), 4, 3.0, 1),
    ((1, 1, 1), 2, 2.0, 0),         # no neighbours: H = F = 0
    ((7, 1, 1), 3, 2.0, 0),         # a line along z
    ((1, 40, 1), 2, 2.0, 1),
    ((1, 96, 97), 4, 2.0, 0),       # 2D, 8-neighbourhood (k_step_2d)
    ((1, 70, 130), 3, 1.5, 1),      # 2D, several tiles, ragged, general m
    ((1, 140, 41), 4, 2.0, 0),      # 2D, 9 tile rows: CTA columns of 4 + 4 + 1 tiles
]


@pytest.mark.parametrize("shape,C,m,q_mode", CASES)
def test_step_parity(ctx, orc, shape, C, m, q_mode):
    nz, ny, nx = shape
    states = [random_state(nx, ny, nz, C, seed=100 + s, crisp_frac=0.1) for s in range(3)]
    x = states[0][0]
    Us = [s[1] for s in states]
    cs = [s[2] for s in states]
    lamxi = [(0.3, 0.6), (1.0, 1.0), (0.05, 0.95)]
    U, c, st = gpu_step(ctx, x, Us, cs, lamxi, C, m=m, q_mode=q_mode)
    for p in range(3):
        Uo, co, Jo, duo = orc.ifcm_step(x, Us[p], cs[p], *lamxi[p], m=m, q_mode=q_mode)
        err = np.abs(U[p] - Uo).max()
        assert err < U_TOL, (p, err)
        assert np.all(np.abs(c[p] - co) <= C_TOL * np.abs(co) + 1e-7), (c[p], co)
        assert abs(st[p, 0] - Jo) <= 1e-4 * abs(Jo) + 1e-9, (st[p, 0], Jo)
        assert abs(st[p, 1] - duo) < 2e-4
        assert np.abs(U[p].sum(1) - 1).max() < 1e-5


@pytest.mark.parametrize("shape,C,m,q_mode", [
    ((9, 17, 33), 4, 2.0, 0),
    ((19, 37, 70), 4, 2.0, 1),
    ((17, 16, 32), 3, 1.5, 0),
    ((1, 70, 130), 4, 2.0, 0),      # 2D kernel
])
def test_step_parity_offgrid_x(ctx, orc, shape, C, m, q_mode):
    """Intensities off the u8 grid (fp32 values of an f32 volume's
    normalisation, random in [0, 1)): the same 1e-4 / 1e-4 bounds, one step
    and three chained steps (3e-4, the per-step bound compounded)."""
    nz, ny, nx = shape
    states = [random_state(nx, ny, nz, C, seed=500 + s, u8_levels=False, crisp_frac=0.1) for s in range(3)]
    x = states[0][0]
    assert not np.allclose(x * 255, np.round(x * 255))
    Us = [s[1] for s in states]
    cs = [s[2] for s in states]
    lamxi = [(0.3, 0.6), (1.0, 1.0), (0.05, 0.95)]
    U, c, st = gpu_step(ctx, x, Us, cs, lamxi, C, m=m, q_mode=q_mode)
    for p in range(3):
        Uo, co, Jo, _ = orc.ifcm_step(x, Us[p], cs[p], *lamxi[p], m=m, q_mode=q_mode)
        assert np.abs(U[p] - Uo).max() < U_TOL, p
        assert np.all(np.abs(c[p] - co) <= C_TOL * np.abs(co) + 1e-7), (c[p], co)
        assert abs(st[p, 0] - Jo) <= 1e-4 * abs(Jo) + 1e-9
    U3, c3, _ = gpu_step(ctx, x, Us[:1], cs[:1], lamxi[:1], C, m=m, q_mode=q_mode, iters=3)
    Uo, co = Us[0].astype(np.float64), cs[0].astype(np.float64)
    for _ in range(3):
        Uo, co, _, _ = orc.ifcm_step(x, Uo, co, *lamxi[0], m=m, q_mode=q_mode)
    assert np.abs(U3[0] - Uo).max() < 3e-4


CASES_V2 = [
    # (nz, ny, nx), C, m, q_mode, h -- two Chebyshev shells (NEXT-2, Eq. 10)
    ((1, 9, 9), 2, 2.0, 0, 1.0),
    ((6, 13, 14), 3, 2.0, 0, 1.0),
    ((11, 21, 37), 4, 2.0, 1, 0.5),     # ragged tiles in x and y, z chunk tails
    ((20, 33, 66), 4, 2.0, 0, 2.0),     # several tiles in every direction
    ((5, 3, 40), 4, 1.5, 0, 1.0),       # thin in y: boundary Qs everywhere
    ((2, 2, 2), 2, 2.0, 1, 1.0),        # every voxel sees the whole volume
]


CASES_V3 = [
    # (nz, ny, nx), C, m, q_mode, h -- three Chebyshev shells (342 neighbours)
    ((1, 11, 12), 2, 2.0, 0, 1.0),      # 2D
    ((9, 21, 37), 4, 2.0, 0, 1.0),      # ragged tiles, boundary shells everywhere
    ((14, 40, 70), 3, 2.0, 1, 0.7),     # several tiles, interior voxels
    ((3, 3, 3), 4, 1.5, 0, 2.0),        # every voxel sees the whole volume
]


@pytest.mark.parametrize("v,shape,C,m,q_mode,h", [(2,) + c for c in CASES_V2] + [(3,) + c for c in CASES_V3])
def test_step_parity_v2(ctx, orc, v, shape, C, m, q_mode, h):
    """v = 2, 3 (Eq. 9-10): every membership within 1e-4, centres
    1e-4 relative, J 1e-4."""
    nz, ny, nx = shape
    states = [random_state(nx, ny, nz, C, seed=300 + s, crisp_frac=0.1) for s in range(3)]
    x = states[0][0]
    Us = [s[1] for s in states]
    cs = [s[2] for s in states]
    lamxi = [(0.3, 0.6), (1.0, 1.0), (0.05, 0.95)]
    U, c, st = gpu_step(ctx, x, Us, cs, lamxi, C, m=m, q_mode=q_mode, v=v, h=h)
    for p in range(3):
        Uo, co, Jo, duo = orc.ifcm_step(x, Us[p], cs[p], *lamxi[p], m=m, q_mode=q_mode, v=v, h=h)
        err = np.abs(U[p] - Uo).max()
        assert err < U_TOL, (p, err)
        assert np.all(np.abs(c[p] - co) <= C_TOL * np.abs(co) + 1e-7), (c[p], co)
        assert abs(st[p, 0] - Jo) <= 1e-4 * abs(Jo) + 1e-9, (st[p, 0], Jo)
        assert np.abs(U[p].sum(1) - 1).max() < 1e-5


def test_v2_multi_iteration_and_pso(ctx, orc):
    """v = 2 over 5 iterations from the same start (1e-4 per iteration is
    compounded; checked at 5e-4) and the CHAINED PSO eval (generation 0
    fitness within 1e-5)."""
    from paper_2002_01981_b200 import IfcmConfig, PsoConfig, to_aos, to_pitched_x
    from paper_2002_01981_b200.api import _grid
    nz, ny, nx, C = 8, 20, 24, 3
    x, U0, c0 = random_state(nx, ny, nz, C, seed=41, crisp_frac=0.1)
    U, c, st = gpu_step(ctx, x, [U0], [c0], [(0.4, 0.5)], C, iters=5, v=2, h=1.0)
    Uo, co = U0.astype(np.float64), c0.astype(np.float64)
    for _ in range(5):
        Uo, co, _, _ = orc.ifcm_step(x, Uo, co, 0.4, 0.5, v=2, h=1.0)
    assert np.abs(U[0] - Uo).max() < 5e-4
    dev = torch.device("cuda:0")
    cfg = IfcmConfig(C=C, v=2, h=1.0)
    pso = PsoConfig(P=5, max_gen=2, patience=0, seed=9)
    ws = ctx.workspace(nx, ny, nz, cfg, pso)
    g = _grid(nx, ny, nz)
    c4 = torch.zeros(4, device=dev)
    c4[:C] = torch.as_tensor(c0)
    ctx.pso_init(g, cfg, pso, to_aos(U0, dev), c4, ws)
    ctx.pso_eval(g, cfg, pso, to_pitched_x(x, dev), ws)
    f = ctx.pso_fitness(g, cfg, pso, ws).cpu().numpy()
    r = orc.pso_run(x, U0, c0, P=5, max_gen=1, seed=9, v=2, h=1.0)
    assert np.allclose(f, r.trace_f[0], rtol=1e-5, atol=0)


def test_fcm_pointwise_parity(ctx, orc):
    """lambda = xi = 0 for every state -> the pointwise (FCM) kernel; equals the
    oracle's independent FCM step (PAPER:61 with lambda = xi = 0)."""
    x, U0, c0 = random_state(45, 31, 6, 4, seed=7)
    U, c, st = gpu_step(ctx, x, [U0, U0], [c0, c0 + 0.01], [(0, 0), (0, 0)], 4)
    for p, cc in enumerate([c0, c0 + 0.01]):
        Uf, cf, Jf, _ = orc.fcm_step(x, cc.astype(np.float32).astype(np.float64))
        assert np.abs(U[p] - Uf).max() < U_TOL
        assert np.all(np.abs(c[p] - cf) <= C_TOL * np.abs(cf))
        assert abs(st[p, 0] - Jf) <= 1e-4 * Jf


def test_multi_iteration_and_convergence(ctx, orc):
    from inputs import cube_phantom, add_noise_u8
    img, _ = cube_phantom(40, 36, 12, (0.1, 0.5, 0.9))
    x = (add_noise_u8(img, 7.0, 5).astype(np.float32) / 255.0)
    Uf, cf, _ = orc.fcm_run(x, np.array([0.1, 0.5, 0.9]), max_iter=3)
    U0 = Uf.astype(np.float32)
    c0 = cf.astype(np.float32)
    U5, c5, st = gpu_step(ctx, x, [U0], [c0], [(0.4, 0.7)], 3, iters=5)
    Uo, co, it, _ = orc.ifcm_run(x, U0, c0, 0.4, 0.7, eps=0.0, max_iter=5)
    assert np.abs(U5[0] - Uo).max() < 5 * U_TOL
    assert np.all(np.abs(c5[0] - co) <= 5 * C_TOL * co)
    assert st[0, 2] == 5
    # with eps: stops early and the result equals running exactly that many iterations
    Ue, ce, ste = gpu_step(ctx, x, [U0], [c0], [(0.4, 0.7)], 3, iters=60, eps=1e-3)
    k = int(ste[0, 2])
    assert ste[0, 3] == 1 and 1 <= k < 60 and ste[0, 1] < 1e-3
    Uk, ck, _ = gpu_step(ctx, x, [U0], [c0], [(0.4, 0.7)], 3, iters=k)
    assert (Ue == Uk).all() and (ce == ck).all()


def test_determinism(ctx):
    x, U0, c0 = random_state(70, 40, 20, 4, seed=3)
    a = gpu_step(ctx, x, [U0, U0], [c0, c0], [(0.2, 0.9), (0.7, 0.1)], 4, iters=2)
    b = gpu_step(ctx, x, [U0, U0], [c0, c0], [(0.2, 0.9), (0.7, 0.1)], 4, iters=2)
    for u, v in zip(a, b):
        assert (u == v).all()


def test_constant_volume_and_crisp(ctx, orc):
    """R3: constant intensities -> G = 0 -> H = 0; R5: x == c -> crisp rows."""
    x = np.full((4, 9, 10), 100 / 255, np.float32)
    _, U0, _ = random_state(10, 9, 4, 3, seed=1)
    c0 = np.array([0.1, 100 / 255, 0.9], np.float32)
    U, c, st = gpu_step(ctx, x, [U0], [c0], [(1.0, 0.5)], 3)
    assert (U[0] == np.array([0.0, 1.0, 0.0])).all()
    c1 = np.array([0.1, 0.5, 0.9], np.float32)
    U, c, st = gpu_step(ctx, x, [U0], [c1], [(1.0, 0.5)], 3)
    Uo, _, _, _ = orc.ifcm_step(x, U0, c1, 1.0, 0.5)
    assert np.abs(U[0] - Uo).max() < U_TOL


def test_argmax_bit_exact(ctx, orc):
    """Defuzzification (R13) is bit-exact given identical memberships,
    including exact ties (lowest index wins)."""
    from paper_2002_01981_b200 import to_aos
    rng = np.random.default_rng(0)
    nz, ny, nx = 6, 11, 13
    U = rng.integers(0, 4, size=(nz * ny * nx, 4)).astype(np.float32) / 4  # many ties
    for C in (2, 3, 4):
        Ut = to_aos(U[:, :C], torch.device("cuda:0"))
        lab = ctx.argmax(Ut, nx, ny, nz, C).cpu().numpy().ravel()
        assert (lab == orc.argmax(U[:, :C].astype(np.float64))).all()


def test_normalize_hist_gmm(ctx, orc):
    from inputs import config_volume
    vol, _ = config_volume("C3", shape=(20, 26, 23))
    vt = torch.as_tensor(vol, device="cuda:0")
    x, hist = ctx.normalize_u8(vt)
    xo = orc.normalize_u8(vol)
    xg = x[:, :, :23].cpu().numpy()
    assert np.abs(xg - xo).max() <= 6e-8
    assert (x[:, :, 23:] == 0).all()
    assert (hist.cpu().numpy() == orc.histogram_u8(vol)).all()
    c0 = ctx.gmm_init(hist, 4).cpu().numpy()[:4]
    co = orc.gmm_init(orc.histogram_u8(vol), 4)
    assert np.abs(c0 - co).max() < 1e-6


def test_error_codes(ctx):
    from paper_2002_01981_b200 import IfcmConfig, PifcmError
    dev = torch.device("cuda:0")
    x = torch.zeros((2, 4, 4), device=dev)
    U = torch.zeros((1, 32, 4), device=dev)
    cen = torch.zeros((1, 4), device=dev)
    lx = torch.zeros((1, 2), dtype=torch.float64, device=dev)
    with pytest.raises(PifcmError) as e:
        ctx.iterate(x, U, U, cen, lx, IfcmConfig(C=3), nx=4)
    assert e.value.code == -1
    with pytest.raises(PifcmError) as e:
        ctx.iterate(x, U, torch.zeros_like(U), cen, lx, IfcmConfig(C=5), nx=4)
    assert e.value.code == -1


def test_same_state_parity_ill_conditioned(ctx, orc):
    """At lambda = xi = 1 the Eq. 4 factor approaches 0 on mixed boundaries and
    u becomes proportional to it (condition number u(1-u)/a).  Iterating the
    GPU state 30 times and checking every iteration from the GPU's own previous
    state keeps the 1e-4 bound (the fp64 re-evaluation band)."""
    from inputs import cube_phantom, add_noise_u8
    from paper_2002_01981_b200 import IfcmConfig, to_aos, to_pitched_x
    img, _ = cube_phantom(24, 20, 8, (0.1, 0.5, 0.9))
    x = add_noise_u8(img, 7.0, 3).astype(np.float32) / 255.0
    Uf, cf, _ = orc.fcm_run(x, np.array([0.1, 0.5, 0.9]))
    dev = torch.device("cuda:0")
    Ut = to_aos(Uf.astype(np.float32), dev).view(1, -1, 4)
    Uo = torch.empty_like(Ut)
    cen = torch.zeros(1, 4, device=dev)
    cen[0, :3] = torch.as_tensor(cf.astype(np.float32))
    lx = torch.tensor([[1.0, 1.0]], dtype=torch.float64, device=dev)
    xt = to_pitched_x(x, dev)
    worst = 0.0
    for it in range(30):
        pu = Ut[0, :, :3].cpu().numpy().astype(np.float64)
        pc = cen[0, :3].cpu().numpy().astype(np.float64)
        ctx.iterate(xt, Ut, Uo, cen, lx, IfcmConfig(C=3), nx=24)
        Us, cs, _, _ = orc.ifcm_step(x, pu, pc, 1.0, 1.0)
        err = np.abs(Uo[0, :, :3].cpu().numpy() - Us).max()
        worst = max(worst, err)
        assert err < U_TOL, (it, err)
        assert np.all(np.abs(cen[0, :3].cpu().numpy() - cs) <= C_TOL * np.abs(cs) + 1e-7)
        Ut, Uo = Uo, Ut


@pytest.mark.parametrize("shape,C,m,q_mode", [((1, 32, 32), 3, 2.0, 0), ((1, 50, 40), 4, 1.7, 1), ((1, 7, 61), 2, 2.0, 0)])
def test_small2d_multi_iteration(ctx, orc, shape, C, m, q_mode):
    """pifcm_iterate on a small 2D image runs every iteration in one launch
    (small2d.cu): one iteration from the same state within 1e-4 for three
    states at once; six iterations against the oracle's run (1e-3, as C1);
    the eps stop at the oracle's iteration count."""
    from paper_2002_01981_b200 import IfcmConfig, to_aos, to_pitched_x
    nz, ny, nx = shape
    dev = torch.device("cuda:0")
    states = [random_state(nx, ny, nz, C, seed=500 + s, crisp_frac=0.05) for s in range(3)]
    x = states[0][0]
    lams = [(0.3, 0.6), (0.8, 0.9), (0.0, 0.0)]
    U = torch.stack([to_aos(s[1], dev) for s in states])
    cen = torch.zeros((3, 4), device=dev)
    for i, s in enumerate(states):
        cen[i, :C] = torch.as_tensor(s[2])
    lx = torch.tensor(lams, dtype=torch.float64, device=dev)
    xt = to_pitched_x(x, dev)
    Un = torch.empty_like(U)
    stats = torch.zeros((3, 4), dtype=torch.float64, device=dev)
    c1 = cen.clone()
    ctx.iterate(xt, U, Un, c1, lx, IfcmConfig(C=C, m=m, q_mode=q_mode, eps=0.0), iters=1, stats=stats, nx=nx)
    for i, s in enumerate(states):
        Uo, co, Jo, _ = orc.ifcm_step(x, s[1], s[2], lams[i][0], lams[i][1], m=m, q_mode=q_mode)
        assert np.abs(Un[i, :, :C].cpu().numpy() - Uo).max() < 1e-4, i
        assert np.allclose(c1[i, :C].cpu().numpy(), co, rtol=1e-4)
        assert abs(stats[i, 0].item() - Jo) <= 1e-4 * Jo
    c6 = cen.clone()
    ctx.iterate(xt, U, Un, c6, lx, IfcmConfig(C=C, m=m, q_mode=q_mode, eps=0.0), iters=6, stats=stats, nx=nx)
    assert (stats[:, 2].cpu().numpy() == 6).all()
    for i, s in enumerate(states):
        Ur, cr, it, _ = orc.ifcm_run(x, s[1], s[2], lams[i][0], lams[i][1], eps=0.0, max_iter=6, m=m, q_mode=q_mode)
        assert np.abs(Un[i, :, :C].cpu().numpy() - Ur).max() < 1e-3, i
    ce = cen.clone()
    ctx.iterate(xt, U, Un, ce, lx, IfcmConfig(C=C, m=m, q_mode=q_mode, eps=1e-3), iters=100, stats=stats, nx=nx)
    for i, s in enumerate(states):
        _, _, it, _ = orc.ifcm_run(x, s[1], s[2], lams[i][0], lams[i][1], eps=1e-3, max_iter=100, m=m, q_mode=q_mode)
        assert abs(int(stats[i, 2].item()) - it) <= 1, (i, stats[i, 2].item(), it)


@pytest.mark.parametrize("shape,iters,eps", [((96, 97), 20, 0.0), ((140, 41), 30, 1e-4), ((854, 854), 12, 0.0)])
def test_2d_cooperative_loop_equals_per_step(ctx, shape, iters, eps):
    """The final IFCM of a 2D image in one cooperative launch
    (k_step_2d_loop: grid barriers, canonical finalisation by CTA 0) against
    one launch per iteration: memberships, centres and stats bit-identical,
    including an eps stop before the last iteration."""
    from paper_2002_01981_b200 import IfcmConfig, to_aos, to_pitched_x
    ny, nx = shape
    x, U, c = random_state(nx, ny, 1, 4, seed=5, crisp_frac=0.1)
    dev = torch.device("cuda:0")
    xt = to_pitched_x(x, dev)
    cfg = IfcmConfig(C=4, eps=eps)
    lx = torch.tensor([[0.7, 0.9]], dtype=torch.float64, device=dev)
    out = []
    for per_step in (True, False):
        Ui = to_aos(U, dev).view(1, -1, 4)
        Uo = torch.empty_like(Ui)
        cen = torch.zeros((1, 4), device=dev)
        cen[0, :4] = torch.as_tensor(c)
        st = torch.zeros((1, 4), dtype=torch.float64, device=dev)
        ctx.iterate(xt, Ui, Uo, cen, lx, cfg, iters=iters, stats=st, nx=nx, canonical=True, per_step=per_step)
        out.append((Uo.clone(), cen.clone(), st.clone()))
    (U1, c1, s1), (U2, c2, s2) = out
    assert torch.equal(U1, U2) and torch.equal(c1, c2) and torch.equal(s1, s2), (s1, s2)
    if eps > 0:
        assert 1 <= s1[0, 2].item() <= iters
