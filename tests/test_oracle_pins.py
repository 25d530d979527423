"""Pins of the fp64 oracle's IFCM step against what the paper and the
mathematics fix (not against itself).  CPU only.

PAPER:N = /root/reference/PAPER.md line N.
"""
import json
import os

import numpy as np
import pytest

from tests import bruteforce as bf

GOLD = os.path.join(os.path.dirname(__file__), "golden", "worked_example_3x3.json")


def _gold():
    with open(GOLD) as f:
        return json.load(f)


def _ex_state(g):
    x = np.array(g["x"], np.float64)
    u0 = np.array(g["u0"], np.float64).ravel()
    U = np.stack([u0, 1.0 - u0], axis=1)
    return x, U, np.array(g["c"])


# --------------------------------------------------------------------------- worked example
def test_worked_example_centre_by_hand():
    """Centre voxel of the 3x3 example, derived by hand from Eqs. 4-8.

    Neighbours of (1,1): edges (q=1) all have x=0.5 -> g=0; corners (q=2)
    have x in {0,1} -> g=0.5.  G = 4*0.5 = 2; literal q^2: Qs = 4*1 + 4*4 = 20.
    Hn_0 = 0.5*(0.9+0.1+0.2+0.4) = 0.8 -> H_0 = 0.4 (Eq. 5).
    Fn_0 = (.64+.49+.09+.36) + 4*(.81+.01+.04+.16) = 5.66 -> F_0 = 0.283 (Eq. 7).
    a_0 = 1 - .5*.4 - .5*.283 = .6585; d2_0 = .09*.6585 = .059265 (Eq. 4).
    u_0 = (1/d2_0)/(1/d2_0 + 1/d2_1) (Eq. 2, m=2)."""
    g = _gold()
    assert 4 * 0.5 == g["literal"]["centre"]["G"]
    assert 4 * 1 + 4 * 4 == g["literal"]["centre"]["Qs"]
    hn0 = 0.5 * (0.9 + 0.1 + 0.2 + 0.4)
    assert abs(hn0 / 2.0 - 0.4) < 1e-15
    fn0 = (0.64 + 0.49 + 0.09 + 0.36) + 4 * (0.81 + 0.01 + 0.04 + 0.16)
    assert abs(fn0 / 20 - 0.283) < 1e-15
    d2 = g["literal"]["centre"]["d2"]
    u0 = (1 / d2[0]) / (1 / d2[0] + 1 / d2[1])
    assert abs(u0 - g["literal"]["centre"]["u"][0]) < 1e-10


@pytest.mark.parametrize("mode,key", [(0, "literal"), (1, "sqeuclid")])
def test_worked_example_step(orc, mode, key):
    g = _gold()
    x, U, c = _ex_state(g)
    Un, cn, J, _ = orc.ifcm_step(x, U, c, g["lambda"], g["xi"], m=g["m"], q_mode=mode)
    exp = g[key]
    assert np.allclose(Un[4], exp["centre"]["u"], atol=1e-10)
    assert np.allclose(cn, exp["c_new"], atol=1e-10)
    assert abs(J - exp["J"]) < 1e-10
    if key == "literal":
        assert np.allclose(Un[0], exp["voxel00"]["u"], atol=1e-10)
        assert (orc.argmax(Un).reshape(3, 3) == np.array(exp["labels"])).all()
        u, d2, H, F = orc.ifcm_voxels(x, U, c, g["lambda"], g["xi"], [4, 0], q_mode=0)
        assert np.allclose(H[0], exp["centre"]["H"], atol=1e-12)
        assert np.allclose(F[0], exp["centre"]["F"], atol=1e-12)
        assert np.allclose(d2[0], exp["centre"]["d2"], atol=1e-12)
        assert np.allclose(H[1], exp["voxel00"]["H"], atol=1e-12)
        assert np.allclose(F[1], exp["voxel00"]["F"], atol=1e-12)


def test_worked_example_fcm_reduction(orc):
    g = _gold()
    x, U, c = _ex_state(g)
    Un, cn, J, _ = orc.ifcm_step(x, U, c, 0.0, 0.0)
    exp = g["fcm_lambda_xi_zero"]
    assert np.allclose(Un[4], exp["centre"]["u"], atol=1e-12)
    assert orc.argmax(Un)[4] == exp["centre"]["label"]  # tie -> lowest index (R13)
    assert np.allclose(Un[0], exp["voxel00"]["u"], atol=1e-10)
    assert np.allclose(cn, exp["c_new"], atol=1e-10)
    assert abs(J - exp["J"]) < 1e-10


def test_worked_example_bruteforce_agrees():
    g = _gold()
    x, U, c = _ex_state(g)
    for mode, key in ((0, "literal"), (1, "sqeuclid")):
        Un, cn, J, _ = bf.ifcm_step_bruteforce(x, U, c, 0.5, 0.5, q_mode=mode)
        assert np.allclose(cn, g[key]["c_new"], atol=1e-10)
        assert abs(J - g[key]["J"]) < 1e-10


# --------------------------------------------------------------------------- SPEC examples
def test_fcm_textbook_membership(orc):
    """SPEC:147-148 from Eq. 2: x=.25, c={0,1}, m=2 -> (0.9, 0.1); equidistant -> (.5,.5)."""
    U, _, _, _ = orc.fcm_step(np.array([0.25]), np.array([0.0, 1.0]))
    assert np.allclose(U[0], [0.9, 0.1], atol=1e-15)
    U, _, _, _ = orc.fcm_step(np.array([0.5]), np.array([0.25, 0.75]))
    assert np.allclose(U[0], [0.5, 0.5], atol=1e-15)
    U, _, _, _ = orc.fcm_step(np.array([0.75]), np.array([0.25, 0.75, 0.9]))
    assert U[0].tolist() == [0.0, 1.0, 0.0]  # zero distance -> crisp (R5)


def test_centres_textbook(orc):
    """SPEC:156-158 from Eq. 3: crisp -> group means; {0,1}, u=.5, m=2 -> 0.5."""
    x = np.array([0.2, 0.2, 0.8])
    U = np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    assert np.allclose(orc.centers(x, U, [0, 0]), [0.2, 0.8], atol=1e-15)
    x = np.array([0.0, 1.0])
    U = np.array([[0.5, 0.5], [0.5, 0.5]])
    assert abs(orc.centers(x, U, [0, 0])[0] - 0.5) < 1e-15
    # empty cluster keeps its previous centre (R9)
    U = np.array([[1.0, 0.0], [1.0, 0.0]])
    assert orc.centers(x, U, [0.3, 0.7])[1] == 0.7


def test_shell_weights(orc):
    """Eq. 10: W(2,1) = (e^-1, e^-2)/(e^-1+e^-2); W(1,.) = 1."""
    assert np.allclose(orc.shell_weights(2, 1.0), [0.7310585786, 0.2689414214], atol=1e-9)
    assert orc.shell_weights(1, 3.7).tolist() == [1.0]
    rng = np.random.default_rng(0)
    for _ in range(50):
        v = int(rng.integers(1, 8))
        h = float(rng.uniform(0.1, 5))
        W = orc.shell_weights(v, h)
        assert abs(W.sum() - 1) < 1e-12 and (np.diff(W) < 0).all()


def test_single_neighbour_H_and_d2(orc):
    """SPEC:278 H: single neighbour u=.6, g=.3 -> H=.6 (2x1x1 volume)
    d2 = .09*(1 - .5*.6 - .2*.25) = .0585 with F = .25 (q=1, u=.5)."""
    x = np.array([[[0.5, 0.2]]])
    U = np.array([[0.5, 0.5], [0.6, 0.4]])
    u, d2, H, F = orc.ifcm_voxels(x, U, [0.2, 0.9], 0.5, 0.2, [0])
    assert abs(H[0, 0] - 0.6) < 1e-15 and abs(H[0, 1] - 0.4) < 1e-15
    U2 = np.array([[0.5, 0.5], [0.5, 0.5]])
    u, d2, H, F = orc.ifcm_voxels(x, U2, [0.2, 0.9], 0.5, 0.2, [0])
    assert abs(F[0, 0] - 0.25) < 1e-15
    # with H forced to .6 via U: F becomes .36; use the printed combination directly
    u, d2, H, F = orc.ifcm_voxels(x, U, [0.2, 0.9], 0.5, 0.2, [0])
    assert abs(d2[0, 0] - 0.09 * (1 - 0.5 * H[0, 0] - 0.2 * F[0, 0])) < 1e-15
    assert abs(0.09 * (1 - 0.5 * 0.6 - 0.2 * 0.25) - 0.0585) < 1e-15


def test_F_equal_neighbours(orc):
    """Eq. 7 with all neighbour memberships equal to w -> F = w^2 (any q weights)."""
    x = np.zeros((1, 2, 2))
    U = np.full((4, 2), 0.5)
    for mode in (0, 1):
        _, _, _, F = orc.ifcm_voxels(x, U, [0.1, 0.9], 0.3, 0.3, [0, 3], q_mode=mode)
        assert np.allclose(F, 0.25, atol=1e-15)


def test_constant_volume_H_zero(orc):
    """R3: all g = 0 -> H = 0; then with xi = 0 the step is FCM."""
    x = np.full((3, 4, 5), 0.4)
    rng = np.random.default_rng(1)
    U = rng.random((60, 3))
    U /= U.sum(1, keepdims=True)
    _, _, H, _ = orc.ifcm_voxels(x, U, [0.1, 0.5, 0.9], 1.0, 0.0, np.arange(60))
    assert (H == 0).all()


# --------------------------------------------------------------------------- neighbourhood
@pytest.mark.parametrize("dims", [(5, 6, 7), (4, 4, 1), (3, 1, 1), (1, 1, 3)])
def test_neighbour_counts_and_qsum(orc, dims):
    """Eq. 9 counts (interior 26, face 17, edge 11, corner 7; 2D 8/5/3) and the
    Eq. 7 denominators, from brute force over all voxel pairs; checked through
    the oracle with constant U (H = w_j) and U = one-hot neighbour (F = q2/Qs)."""
    nx, ny, nz = dims
    if dims == (5, 6, 7):
        assert bf.neighbour_count_bruteforce(5, 6, 7, 2, 2, 2) == 26
        assert bf.neighbour_count_bruteforce(5, 6, 7, 0, 2, 2) == 17
        assert bf.neighbour_count_bruteforce(5, 6, 7, 0, 0, 2) == 11
        assert bf.neighbour_count_bruteforce(5, 6, 7, 0, 0, 0) == 7
        assert bf.qsum_bruteforce(5, 6, 7, 2, 2, 2, 0) == 126
        assert bf.qsum_bruteforce(5, 6, 7, 2, 2, 2, 1) == 54
        assert bf.qsum_bruteforce(5, 6, 7, 0, 2, 2, 0) == 73
        assert bf.qsum_bruteforce(5, 6, 7, 0, 0, 2, 0) == 42
        assert bf.qsum_bruteforce(5, 6, 7, 0, 0, 0, 0) == 24
    if dims == (4, 4, 1):
        assert bf.neighbour_count_bruteforce(4, 4, 1, 1, 1, 0) == 8
        assert bf.neighbour_count_bruteforce(4, 4, 1, 0, 1, 0) == 5
        assert bf.neighbour_count_bruteforce(4, 4, 1, 0, 0, 0) == 3
        assert bf.qsum_bruteforce(4, 4, 1, 1, 1, 0, 0) == 20
        assert bf.qsum_bruteforce(4, 4, 1, 1, 1, 0, 1) == 12
    # F with a single neighbour having u = 1 in cluster 0 equals q2_k / Qs_i
    N = nx * ny * nz
    rng = np.random.default_rng(2)
    x = np.zeros((nz, ny, nx))
    for trial in range(4):
        i = int(rng.integers(N))
        k = int(rng.integers(N))
        Xi, Yi, Zi = i % nx, (i // nx) % ny, i // (nx * ny)
        Xk, Yk, Zk = k % nx, (k // nx) % ny, k // (nx * ny)
        d = (Xi - Xk) ** 2 + (Yi - Yk) ** 2 + (Zi - Zk) ** 2
        U = np.zeros((N, 2))
        U[:, 1] = 1.0
        U[k] = [1.0, 0.0]
        for mode in (0, 1):
            _, _, _, F = orc.ifcm_voxels(x, U, [0.1, 0.9], 0.0, 0.0, [i], q_mode=mode)
            Qs = bf.qsum_bruteforce(nx, ny, nz, Xi, Yi, Zi, mode)
            if 0 < d < 4:
                q2 = d * d if mode == 0 else d
                assert abs(F[0, 0] - q2 / Qs) < 1e-15
            else:
                assert F[0, 0] == 0.0


# --------------------------------------------------------------------------- brute force
@pytest.mark.parametrize("shape,C,m,mode,seed", [
    ((1, 8, 8), 2, 2.0, 0, 0),
    ((4, 6, 6), 3, 2.0, 0, 1),
    ((5, 12, 12), 4, 2.0, 1, 2),
    ((3, 5, 7), 3, 1.5, 0, 3),
    ((2, 4, 9), 2, 3.0, 1, 4),
])
def test_oracle_equals_bruteforce(orc, shape, C, m, mode, seed):
    """SPEC acceptance 3: step == uncached pairwise reference (Eq. 9
    literal) within 1e-12 on random tiny volumes."""
    from inputs import random_state
    nz, ny, nx = shape
    x, U, c = random_state(nx, ny, nz, C, seed, crisp_frac=0.2)
    lam, xi = 0.7, 0.4
    Un, cn, J, du = orc.ifcm_step(x, U, c, lam, xi, m=m, q_mode=mode)
    Ub, cb, Jb, dub = bf.ifcm_step_bruteforce(x, U.astype(np.float64), c, lam, xi, m=m, q_mode=mode)
    assert np.abs(Un - np.array(Ub)).max() < 1e-12
    assert np.abs(cn - np.array(cb)).max() < 1e-12
    assert abs(J - Jb) < 1e-12 * max(1.0, abs(Jb))
    assert abs(du - dub) < 1e-12


@pytest.mark.parametrize("shape,C,v,h,mode,seed", [((5, 6, 7), 3, 2, 1.0, 0, 3), ((6, 5, 5), 4, 2, 0.5, 1, 4),
                                                   ((1, 9, 8), 2, 2, 2.0, 0, 5), ((7, 4, 6), 4, 3, 1.0, 0, 6)])
def test_oracle_shells_equal_bruteforce(orc, shape, C, v, h, mode, seed):
    """v >= 2 (R2: Chebyshev shells, Eq. 10 weights, per-shell normalisation)
    == the pairwise reference within 1e-12."""
    from inputs import random_state
    nz, ny, nx = shape
    x, U, c = random_state(nx, ny, nz, C, seed, crisp_frac=0.2)
    Un, cn, J, du = orc.ifcm_step(x, U, c, 0.8, 0.6, q_mode=mode, v=v, h=h)
    Ub, cb, Jb, dub = bf.ifcm_step_bruteforce_shells(x, U.astype(np.float64), c, 0.8, 0.6, v, h, q_mode=mode)
    assert np.abs(Un - np.array(Ub)).max() < 1e-12
    assert np.abs(cn - np.array(cb)).max() < 1e-12
    assert abs(J - Jb) < 1e-12 * max(1.0, abs(Jb))


def test_shells_reduce_to_single_shell(orc):
    """v = 1 is W_1 = 1 (Eq. 10): the shell reference at v = 1 equals the
    literal-Eq. 9 reference."""
    from inputs import random_state
    x, U, c = random_state(5, 4, 3, 3, 9)
    a = bf.ifcm_step_bruteforce(x, U.astype(np.float64), c, 0.5, 0.9)
    b = bf.ifcm_step_bruteforce_shells(x, U.astype(np.float64), c, 0.5, 0.9, 1, 1.0)
    assert np.abs(np.array(a[0]) - np.array(b[0])).max() < 1e-14 and abs(a[2] - b[2]) < 1e-14


# --------------------------------------------------------------------------- input types (a0)
def test_typed_normalize_and_histogram(orc):
    """u16 = 257 * u8 normalises and bins exactly like the u8 volume (the
    integer formula scales); f32 closed forms: min -> 0, max -> 1, constant ->
    0 / bin 0, a value at k/255 of the range -> bin k, affine invariance."""
    from inputs import add_noise_u8, cube_phantom
    img, _ = cube_phantom(11, 9, 4, (0.1, 0.5, 0.9))
    v8 = add_noise_u8(img, 9.0, 12)
    v16 = v8.astype(np.uint16) * 257
    assert (orc.normalize(v16) == orc.normalize(v8)).all()
    assert (orc.histogram(v16) == orc.histogram(v8)).all()
    g = np.random.default_rng(5)
    f = (g.random((3, 5, 7)) * 10 - 3).astype(np.float32)
    x = orc.normalize(f)
    assert x.min() == 0.0 and x.max() == 1.0
    assert np.abs(orc.normalize(f * np.float32(4) + np.float32(2)) - x).max() < 1e-6
    lo, hi = float(f.min()), float(f.max())
    probe = np.array([lo, hi] + [lo + (hi - lo) * k / 255 for k in (1, 17, 128, 254)], np.float32).reshape(1, 1, -1)
    h = orc.histogram(np.concatenate([probe, probe], axis=2))
    for k in (0, 255, 1, 17, 128, 254):
        assert h[k] == 2, (k, h[k])
    c = np.full((2, 3, 4), 7.5, np.float32)
    assert (orc.normalize(c) == 0).all() and orc.histogram(c)[0] == c.size


# --------------------------------------------------------------------------- invariants
def _rand_case(seed, shape=(3, 7, 6), C=3):
    from inputs import random_state
    nz, ny, nx = shape
    return random_state(nx, ny, nz, C, seed, crisp_frac=0.1)


@pytest.mark.parametrize("m", [1.5, 2.0, 3.0])
def test_row_sums(orc, m):
    """SPEC acceptance 1: rows of Eq. 2 sum to 1 (fp64: 1e-12)."""
    for seed in range(20):
        x, U, c = _rand_case(seed, C=2 + seed % 3)
        lam, xi = np.random.default_rng(seed).random(2)
        Un, _, _, _ = orc.ifcm_step(x, U, c, lam, xi, m=m)
        assert np.abs(Un.sum(1) - 1).max() < 1e-12
        assert (Un >= 0).all() and (Un <= 1).all()


def test_fcm_reduction(orc):
    """SPEC acceptance 2 / PAPER:61: lambda = xi = 0 reduces Eq. 4 to the plain
    distance, so the step equals the independently written FCM step (1e-12)."""
    for seed in range(30):
        x, U, c = _rand_case(seed, C=2 + seed % 3)
        m = [1.5, 2.0, 3.0][seed % 3]
        Un, cn, J, _ = orc.ifcm_step(x, U, c, 0.0, 0.0, m=m, q_mode=seed % 2)
        Uf, cf, Jf, _ = orc.fcm_step(x, c, m=m)
        assert np.abs(Un - Uf).max() < 1e-12
        assert np.abs(cn - cf).max() < 1e-12
        assert abs(J - Jf) < 1e-12


@pytest.mark.parametrize("m", [1.5, 2.0, 3.0])
def test_cost_closed_form(orc, m):
    """Eq. 1 with Eq. 2 memberships: per voxel sum_j u^m d2 = (sum_j d2^{-1/(m-1)})^{1-m}."""
    x, U, c = _rand_case(5, C=4)
    lam, xi = 0.6, 0.8
    N = U.shape[0]
    _, _, J, _ = orc.ifcm_step(x, U, c, lam, xi, m=m)
    _, d2, _, _ = orc.ifcm_voxels(x, U, c, lam, xi, np.arange(N), m=m)
    Jc = (np.power(d2, -1.0 / (m - 1)).sum(1) ** (1 - m)).sum()
    assert abs(J - Jc) < 1e-10 * Jc


def test_cost_monotone_in_lambda_xi(orc):
    """From a fixed state J is non-increasing in lambda and in xi (H, F >= 0 make
    every d2 non-increasing, and the per-voxel closed form is increasing in d2)."""
    x, U, c = _rand_case(7, shape=(4, 6, 6), C=3)
    grid = np.linspace(0, 1, 6)
    Js = np.array([[orc.ifcm_step(x, U, c, l, s)[2] for s in grid] for l in grid])
    assert (np.diff(Js, axis=0) <= 1e-15).all()
    assert (np.diff(Js, axis=1) <= 1e-15).all()


def test_fcm_cost_descent(orc):
    """the FCM cost sequence is non-increasing (Bezdek's descent).  J of
    step t is evaluated at (U_t, c_{t-1}); the sequence J(U_t, c_t) is what
    descends, so re-evaluate it with the next step's J."""
    from inputs import cube_phantom, add_noise_u8
    img, _ = cube_phantom(24, 24, 1)
    x = add_noise_u8(img, 7.0, 9).astype(np.float64) / 255.0
    c = np.array([0.2, 0.3, 0.6, 0.8])
    Js = []
    for _ in range(15):
        U, c_new, J, _ = orc.fcm_step(x, c)
        Js.append(J)
        c = c_new
    assert (np.diff(Js) <= 1e-12).all()


def test_affine_invariance(orc):
    """Eq. 2-8 are invariant under x -> s x + t, c -> s c + t (g and d scale by
    s; H, F are ratios) : U unchanged, centres transform."""
    x, U, c = _rand_case(11, C=3)
    x = x.astype(np.float64)
    c = c.astype(np.float64)
    s, t = 0.5, 0.25
    Un, cn, J, _ = orc.ifcm_step(x, U, c, 0.4, 0.6)
    Un2, cn2, J2, _ = orc.ifcm_step(s * x + t, U, s * c + t, 0.4, 0.6)
    assert np.abs(Un - Un2).max() < 1e-12
    assert np.abs(cn2 - (s * cn + t)).max() < 1e-12
    assert abs(J2 - s * s * J) < 1e-12


def test_constant_U_gives_H_w_F_w2(orc):
    """Special case of Eqs. 5/7: U rows all equal to w -> H_ij = w_j where G>0,
    F_ij = w_j^2; holds for every shell count v since sum_r W_r = 1 (Eq. 10)."""
    from inputs import random_state
    x, _, c = random_state(6, 5, 4, 3, 12)
    w = np.array([0.2, 0.3, 0.5])
    U = np.tile(w, (120, 1))
    for v in (1, 2):
        _, _, H, F = orc.ifcm_voxels(x, U, c, 0.5, 0.5, np.arange(120), v=v, h=1.3)
        assert np.abs(H - w).max() < 1e-12
        assert np.abs(F - w * w).max() < 1e-12


def test_noiseless_phantom_crisp(orc):
    """Noiseless phantom with centres at the true levels -> every distance to the
    own level is 0 -> crisp rows (R5) and labels == truth."""
    from inputs import cube_phantom
    img, lab = cube_phantom(16, 16, 4, (0.1, 0.35, 0.65, 0.9))
    U = np.full((img.size, 4), 0.25)
    Un, _, J, _ = orc.ifcm_step(img, U, np.array([0.1, 0.35, 0.65, 0.9]), 0.5, 0.5)
    assert ((Un == 0) | (Un == 1)).all()
    assert (orc.argmax(Un) == lab.ravel()).all()
    assert J == 0.0


def test_argmax_ties(orc):
    U = np.array([[0.5, 0.5], [0.2, 0.8], [0.4, 0.3, ][:2], [0.25, 0.25]])
    assert orc.argmax(U).tolist() == [0, 1, 0, 0]


def test_normalize_and_hist(orc):
    """Alg. 2 step 1 min-max: [10,20,30] -> [0,.5,1]; constant -> 0 (R16)."""
    assert orc.normalize_u8(np.array([10, 20, 30], np.uint8)).tolist() == [0.0, 0.5, 1.0]
    assert orc.normalize_u8(np.array([5, 5, 5], np.uint8)).tolist() == [0.0, 0.0, 0.0]
    v = np.arange(256, dtype=np.uint8)
    assert (orc.histogram_u8(v) == 1).all()
    v = np.array([10, 20, 30, 30], np.uint8)
    h = orc.histogram_u8(v)
    assert h.sum() == 4 and h[0] == 1 and h[255] == 2 and h[128] == 1
