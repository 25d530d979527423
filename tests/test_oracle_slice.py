"""Pins of the oracle's literal slice mode (DESIGN R25; Alg. 1 input z,
PAPER:93, 110, 144): the plane-restricted IFCM step against the whole-volume
step and independent reductions, the slice histogram on the volume's levels,
and the nz = 1 reduction of the slice pipeline to the whole pipeline."""
import numpy as np
import pytest

from inputs import add_noise_u8, cube_phantom, random_state


@pytest.mark.parametrize("shape,t", [((5, 7, 6), 0), ((5, 7, 6), 2), ((5, 7, 6), 4), ((2, 9, 8), 1),
                                     ((3, 6, 11), 1)])
def test_step_planes_is_the_whole_step_on_the_target(orc, shape, t):
    nz, ny, nx = shape
    x, U, c = random_state(nx, ny, nz, 4, seed=7 + t, crisp_frac=0.1)
    lam, xi = 0.7, 0.45
    Uw, _, _, _ = orc.ifcm_step(x, U, c, lam, xi)
    Un, cn, J, du = orc.ifcm_step_planes(x, U, c, lam, xi, t, t + 1)
    pl = nx * ny
    tgt = slice(t * pl, (t + 1) * pl)
    # the target plane's rows are the whole step's rows, bit for bit; the
    # other planes are untouched neighbours
    assert (Un[tgt] == Uw[tgt]).all()
    rest = np.ones(U.shape[0], bool)
    rest[tgt] = False
    assert (Un[rest] == U[rest]).all()
    # Eq. 3 over the target plane only (orc_centers: an independent routine)
    xt = np.asarray(x, np.float64).reshape(nz, pl)[t]
    assert np.allclose(cn, orc.centers(xt, Uw[tgt], c), rtol=1e-12, atol=0)
    # Eq. 1 over the target plane only, from the per-voxel evaluation
    u, d2, _, _ = orc.ifcm_voxels(x, U, c, lam, xi, np.arange(t * pl, (t + 1) * pl))
    assert abs(J - float(np.sum(u ** 2 * d2))) <= 1e-12 * J
    assert du == pytest.approx(float(np.abs(Uw[tgt] - U[tgt]).max()), rel=0, abs=0)


def test_step_planes_full_range_is_the_step(orc):
    x, U, c = random_state(6, 5, 4, 3, seed=3)
    a = orc.ifcm_step(x, U, c, 0.3, 0.9)
    b = orc.ifcm_step_planes(x, U, c, 0.3, 0.9, 0, 4)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and a[2] == b[2] and a[3] == b[3]


def test_histogram_range(orc):
    g = np.random.default_rng(5)
    v = g.integers(40, 200, size=(3, 17, 19), dtype=np.uint8)
    # the data's own range: the R15 histogram
    assert (orc.histogram_u8_range(v, v.min(), v.max()) == orc.histogram_u8(v)).all()
    # the full u8 range: bin = ((v * 255) + 127) // 255 = v
    assert (orc.histogram_u8_range(v, 0, 255) == np.bincount(v.ravel(), minlength=256)).all()
    # a constant range: everything in bin 0
    h = orc.histogram_u8_range(np.full(10, 7, np.uint8), 7, 7)
    assert h[0] == 10 and h.sum() == 10


def test_slice_mode_of_a_single_plane_is_the_pipeline(orc):
    """nz = 1: the slice is the volume (no neighbour planes), so the slice
    pipeline equals the whole pipeline exactly."""
    img, _ = cube_phantom(26, 22, 1, (0.1, 0.5, 0.9))
    vol = add_noise_u8(img, 7.0, 4)
    r = orc.segment_u8(vol, C=3, P=5, max_gen=4, seed=9)
    s = orc.segment_slice_u8(vol, 0, C=3, P=5, max_gen=4, seed=9)
    assert (s.labels == r.labels[0]).all()
    assert (s.U == r.U).all() and (s.c == r.c).all() and (s.c_init == r.c_init).all()
    assert (s.lam, s.xi, s.J, s.generations, s.final_iters) == (r.lam, r.xi, r.J, r.generations, r.final_iters)


def test_slice_mode_properties(orc):
    """Interior and boundary slices of a small volume: rows on the simplex,
    labels = argmax of the rows, the GMM start from the slice's histogram on
    the volume's levels."""
    img, _ = cube_phantom(20, 18, 7)
    vol = add_noise_u8(img, 9.0, 6)
    for z in (0, 3, 6):
        s = orc.segment_slice_u8(vol, z, C=4, P=4, max_gen=3, seed=2)
        assert s.labels.shape == (18, 20)
        assert np.allclose(s.U.sum(1), 1.0, atol=1e-12)
        assert (s.labels.ravel() == orc.argmax(s.U)).all()
        h = orc.histogram_u8_range(vol[z], vol.min(), vol.max())
        assert np.allclose(s.c_init, orc.gmm_init(h, 4), rtol=0, atol=0)
        assert 0.0 <= s.lam <= 1.0 and 0.0 <= s.xi <= 1.0 and s.generations == 3
    with pytest.raises(ValueError):
        orc.segment_slice_u8(vol, 7, C=4, P=4, max_gen=3, seed=2)


def test_incs_pins(orc):
    """incS (R26): zero for the truth itself under sorted centres, invariant
    under relabelling the clusters together with their centres, and equal to
    a direct count on random labels."""
    g = np.random.default_rng(3)
    truth = g.integers(0, 4, size=500).astype(np.uint8)
    c = np.array([0.1, 0.35, 0.65, 0.9])
    assert orc.incs(truth, truth, c) == 0
    perm = np.array([2, 0, 3, 1])               # cluster j holds class perm[j]
    lab = np.argsort(perm)[truth].astype(np.uint8)
    assert orc.incs(lab, truth, c[perm]) == 0
    lab = g.integers(0, 4, size=500).astype(np.uint8)
    assert orc.incs(lab, truth, c[perm]) == int((perm[lab] != truth).sum())
    # ties: equal centres rank by index
    assert orc.incs(np.array([0, 1], np.uint8), np.array([0, 1], np.uint8), np.array([0.5, 0.5])) == 0


def test_eq11_worked_example(orc):
    """Eq. 11 by hand: 2 sizes x 3 algorithms, alpha = 0.7."""
    q = np.array([[10.0, 30.0, 20.0], [5.0, 5.0, 5.0]])
    t = np.array([[1.0, 3.0, 2.0], [4.0, 2.0, 3.0]])
    J = orc.eq11(q, t, 0.7)
    # size 0: q -> (0, 1, .5), t -> (0, 1, .5); size 1: q constant -> 0, t -> (1, 0, .5)
    want = np.array([(0.0 + 0.3 * 1.0) / 2, (0.7 + 0.3 + 0.0) / 2, (0.35 + 0.15 + 0.15) / 2])
    assert np.allclose(J, want, rtol=0, atol=1e-15)
    assert np.allclose(orc.eq11(q, t, 1.0), [0.0, 0.5, 0.25])


@pytest.mark.parametrize("shape,t", [((7, 9, 8), 3), ((7, 9, 8), 0), ((7, 9, 8), 5)])
def test_step_planes_v2_is_the_whole_step_on_the_target(orc, shape, t):
    """The plane-restricted step with two shells (v = 2, Eq. 9-10) gives the
    whole v = 2 step's rows on the target plane, bit for bit."""
    nz, ny, nx = shape
    x, U, c = random_state(nx, ny, nz, 4, seed=11 + t, crisp_frac=0.1)
    Uw, _, _, _ = orc.ifcm_step(x, U, c, 0.6, 0.8, v=2, h=1.0)
    Un, _, _, _ = orc.ifcm_step_planes(x, U, c, 0.6, 0.8, t, t + 1, v=2, h=1.0)
    pl = nx * ny
    assert (Un[t * pl:(t + 1) * pl] == Uw[t * pl:(t + 1) * pl]).all()


def test_slice_mode_v2_of_a_single_plane_is_the_pipeline(orc):
    """nz = 1 with v = 2: the slice pipeline equals the whole v = 2 pipeline."""
    img, _ = cube_phantom(26, 22, 1, (0.1, 0.5, 0.9))
    vol = add_noise_u8(img, 7.0, 4)
    r = orc.segment_u8(vol, C=3, P=4, max_gen=3, seed=9, v=2)
    s = orc.segment_slice_u8(vol, 0, C=3, P=4, max_gen=3, seed=9, v=2)
    assert (s.labels == r.labels[0]).all() and (s.U == r.U).all()
    assert (s.lam, s.xi, s.J, s.final_iters) == (r.lam, r.xi, r.J, r.final_iters)


@pytest.mark.parametrize("v", [1, 2])
def test_slice_mode_reads_planes_within_v(orc, v):
    """The slice mode of radius v depends on planes z - v .. z + v only
    (Eq. 9): changing the planes beyond leaves every output identical,
    changing a plane at distance v does not."""
    img, _ = cube_phantom(18, 16, 9, (0.1, 0.35, 0.65, 0.9))
    vol = add_noise_u8(img, 9.0, 3)
    z = 4
    kw = dict(C=4, P=4, max_gen=3, seed=5, v=v)
    s = orc.segment_slice_u8(vol, z, **kw)
    far = vol.copy()
    g = np.random.default_rng(1)
    lo, hi = int(vol.min()), int(vol.max())
    for k in range(9):
        if abs(k - z) > v:  # new values inside the volume's range (Alg. 2 step 1 unchanged)
            far[k] = g.integers(lo, hi + 1, size=far[k].shape, dtype=np.uint8)
    far[0, 0, 0], far[8, 0, 0] = lo, hi
    assert far.min() == lo and far.max() == hi
    f = orc.segment_slice_u8(far, z, **kw)
    assert (f.labels == s.labels).all() and (f.U == s.U).all() and f.J == s.J
    near = vol.copy()
    near[z + v] = 255 - near[z + v]
    n = orc.segment_slice_u8(near, z, **kw)
    assert not (n.U == s.U).all()
