"""Pins of the oracle parts the round-1 review found loosely pinned:

* the GMM start (R15; "Modified_FCM with Gaussian mixture
  model"): every EM iteration -- E step, M-step means, variances and weights
  -- against scikit-learn's GaussianMixture, an independent library
  implementation of the same EM, run from the same start on the histogram
  expanded to samples;
* the swarm initialisation (Alg. 1 step 3; R12): the first
  particles' positions and velocities assembled by hand from the
  KAT-verified Philox4x32-10 words (counter layout, word order, key order,
  the 53-bit double and the velocity map);
* the ring lbest of Alg. 1 step 6 (R12/R13): a worked P = 5,
  k = 1 example with ties whose lbest indices are derived by hand.

CPU only."""
import numpy as np
import pytest


# --------------------------------------------------------------------------
# GMM EM (R15) vs scikit-learn


def _sk_means(hist, C, iters):
    """scikit-learn EM from R15's start: mu_j = (j + 0.5)/C, sigma_j^2 =
    1/(4 C^2), w_j = 1/C, on the samples y_b = b/255 repeated hist[b] times,
    no covariance regularisation, exactly `iters` EM iterations."""
    import warnings

    from sklearn.exceptions import ConvergenceWarning
    from sklearn.mixture import GaussianMixture

    y = np.repeat(np.arange(256) / 255.0, hist).reshape(-1, 1)
    gm = GaussianMixture(n_components=C, covariance_type="spherical", max_iter=iters, tol=0.0,
                         reg_covar=0.0, n_init=1,
                         weights_init=np.full(C, 1.0 / C),
                         means_init=((np.arange(C) + 0.5) / C).reshape(-1, 1),
                         precisions_init=np.full(C, 4.0 * C * C))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", ConvergenceWarning)
        gm.fit(y)
    return np.sort(gm.means_.ravel()), gm


@pytest.mark.parametrize("C,bins,counts", [
    (2, [40, 90, 200], [5, 3, 7]),
    (3, [10, 60, 61, 128, 200, 250], [4, 9, 2, 6, 8, 3]),
    (4, [0, 30, 80, 81, 140, 190, 230, 255], [7, 2, 5, 5, 9, 4, 6, 1]),
])
@pytest.mark.parametrize("iters", [1, 2, 5])
def test_gmm_em_matches_sklearn(orc, C, bins, counts, iters):
    """Iteration 1 pins the E step and the mean update; iterations 2 and 5
    depend on the variance and weight updates of the previous M steps, so a
    wrong variance (e.g. around the old mean), a dropped weight or a wrong
    density normalisation fails here."""
    hist = np.zeros(256, np.int64)
    hist[bins] = counts
    got = orc.gmm_init(hist, C, max_iter=iters)
    want, _ = _sk_means(hist, C, iters)
    # sklearn sums in log space in another order; EM amplifies rounding
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 if iters == 1 else 1e-8)


def test_gmm_em_iterations_matter(orc):
    """The pins above are not vacuous: on these histograms iteration 2 moves
    the means (so variances and weights enter), and the converged fit differs
    from the first iteration."""
    hist = np.zeros(256, np.int64)
    hist[[10, 60, 61, 128, 200, 250]] = [4, 9, 2, 6, 8, 3]
    m1, m2, m50 = (orc.gmm_init(hist, 3, max_iter=k) for k in (1, 2, 50))
    assert np.abs(m1 - m2).max() > 1e-4 and np.abs(m2 - m50).max() > 1e-6


def test_gmm_em_hand_iteration(orc):
    """One EM iteration by hand (C = 2, two bins): bins y = 0 and y = 1, one
    voxel each, start mu = (1/4, 3/4), sigma^2 = 1/16, w = 1/2.  For y = 0
    the distances are d0 = 1/4, d1 = 3/4, so p1/p0 = exp(-(d1^2 - d0^2)/(2 s2))
    = exp(-(9/16 - 1/16) * 8) = e^-4 and the responsibility of component 0 is
    r = 1/(1 + e^-4); y = 1 is the mirror image (responsibility 1 - r).
    M step: mu_0 = (r*0 + (1-r)*1)/(r + 1 - r) = e^-4/(1 + e^-4), mu_1 = 1 - mu_0."""
    hist = np.zeros(256, np.int64)
    hist[0] = 1
    hist[255] = 1
    got = orc.gmm_init(hist, 2, max_iter=1)
    e = np.exp(-4.0)
    assert abs(got[0] - e / (1 + e)) < 1e-15
    assert abs(got[1] - 1.0 / (1 + e)) < 1e-15


# --------------------------------------------------------------------------
# Swarm initialisation (Alg. 1 step 3, R12)


def _u01(w_lo, w_hi):
    return float(((int(w_hi) << 32) | int(w_lo)) >> 11) / 2.0 ** 53


@pytest.mark.parametrize("seed", [0, 12345, 0x0000000200000007])
def test_pso_init_by_hand(orc, seed):
    """x_p = the two 53-bit doubles of Philox(ctr = (0xFFFFFFFF, p, 1, 0),
    key = (seed lo, seed hi)); v_p = (2 u - 1) v0 from ctr (0xFFFFFFFF, p, 2, 0).
    A swapped counter word, key half, word pair or sign fails."""
    v0 = 0.1
    pos, vel = orc.pso_init(3, seed, v0=v0)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for p in range(3):
        o = orc.philox4x32_10([0xFFFFFFFF, p, 1, 0], key)
        assert pos[p, 0] == _u01(o[0], o[1]) and pos[p, 1] == _u01(o[2], o[3])
        o = orc.philox4x32_10([0xFFFFFFFF, p, 2, 0], key)
        assert vel[p, 0] == (2.0 * _u01(o[0], o[1]) - 1.0) * v0
        assert vel[p, 1] == (2.0 * _u01(o[2], o[3]) - 1.0) * v0


def test_pso_init_seed0_particle0_value(orc):
    """The numbers themselves for seed 0, particle 0 (from the Random123
    round function applied to ctr (0xFFFFFFFF, 0, 1, 0), key 0), so that a
    wrong Philox would also show: x_0 in [0,1)^2 and the draws differ from
    the KAT counter-0 words (a counter ignored would reproduce those)."""
    pos, _ = orc.pso_init(1, 0)
    kat0 = _u01(0x6627E8D5, 0xE169C58D)
    assert 0.0 <= pos[0, 0] < 1.0 and pos[0, 0] != kat0


# --------------------------------------------------------------------------
# Ring lbest (Alg. 1 step 6, R12 / R13)


def test_ring_lbest_worked_example(orc):
    """P = 5, ring k = 1, pbest fitness after this generation
        f = [3, 1, 1, 2, 3]      (particles 1 and 2 tie)
    ring neighbourhoods {p-1, p, p+1} mod 5 and their lbest (ties -> lowest
    particle index, R13):
        p=0: {4, 0, 1} -> 1     p=1: {0, 1, 2} -> 1 (tie 1/2 -> 1)
        p=2: {1, 2, 3} -> 1     p=3: {2, 3, 4} -> 2
        p=4: {3, 4, 0} -> 3
    With every pbest at the current position except particle p's own, the
    new velocity of p is v + p1 (pbest_p - x_p) + p2 (x_lbest - x_p); the
    draws (p1, p2) are Philox(ctr = (gen, p, 0, 0), key = seed)."""
    P, gen, seed = 5, 3, 99
    pos = np.array([[0.1, 0.2], [0.3, 0.9], [0.5, 0.5], [0.7, 0.1], [0.95, 0.6]])
    vel = np.zeros((P, 2))
    pbest_f = np.full(P, np.inf)
    pbest_x = pos.copy()
    f = np.array([3.0, 1.0, 1.0, 2.0, 3.0])
    x0 = pos.copy()
    g, imp = orc.pso_update(f, pos, vel, pbest_f, pbest_x, -1, gen, seed, ring_k=1, vmax=10.0)
    assert g == 1 and imp == 1                       # gbest: lowest index of the tie
    lb = [1, 1, 1, 2, 3]
    for p in range(P):
        p1, p2 = orc.philox_pair(seed, gen, p, 0, 0)
        v = p1 * (x0[p] - x0[p]) + p2 * (x0[lb[p]] - x0[p])
        np.testing.assert_array_equal(vel[p], v)
        np.testing.assert_array_equal(pos[p], np.clip(x0[p] + v, 0.0, 1.0))


def test_ring_lbest_k2_wraps(orc):
    """k = 2 on P = 5 covers the whole ring: every lbest is the gbest (index 3
    here, the strict minimum), so the ring reading and the gbest topology
    agree; with k = 1 particle 0 ({4, 0, 1}) must not see particle 3."""
    P, gen, seed = 5, 0, 7
    pos = np.array([[0.2, 0.2], [0.4, 0.4], [0.6, 0.6], [0.8, 0.8], [0.9, 0.1]])
    f = np.array([5.0, 4.0, 3.0, 1.0, 2.0])
    for k, lb0 in ((2, 3), (1, 4)):
        p_ = pos.copy()
        vel = np.zeros((P, 2))
        pbf = np.full(P, np.inf)
        orc.pso_update(f, p_, vel, pbf, pos.copy(), -1, gen, seed, ring_k=k, vmax=10.0)
        p1, p2 = orc.philox_pair(seed, gen, 0, 0, 0)
        np.testing.assert_array_equal(vel[0], p2 * (pos[lb0] - pos[0]))


def test_gbest_incumbent_keeps_exact_tie(orc):
    """R13: the gbest is the lowest index among the minimal pbests, but the
    incumbent keeps it on an exact tie -- its evaluation's state is the
    pinned snapshot (Alg. 1 step 10) and a tied particle did not
    improve on it.  Worked example, P = 4:
        generation 0: f = [5, 4, 2, 3]  -> gbest 2 (strict minimum), improved
        generation 1: f = [2, 9, 9, 9]  -> particle 0 ties the incumbent's 2:
                                           gbest stays 2, not improved
        generation 2: f = [1, 9, 9, 9]  -> particle 0 is strictly better:
                                           gbest 0, improved"""
    P, seed = 4, 5
    pos = np.array([[0.1, 0.1], [0.3, 0.3], [0.5, 0.5], [0.7, 0.7]])
    vel = np.zeros((P, 2))
    pbf = np.full(P, np.inf)
    pbx = pos.copy()
    g, imp = orc.pso_update(np.array([5.0, 4.0, 2.0, 3.0]), pos, vel, pbf, pbx, -1, 0, seed)
    assert (g, imp) == (2, 1)
    g, imp = orc.pso_update(np.array([2.0, 9.0, 9.0, 9.0]), pos, vel, pbf, pbx, g, 1, seed)
    assert (g, imp) == (2, 0) and pbf[0] == pbf[2] == 2.0
    g, imp = orc.pso_update(np.array([1.0, 9.0, 9.0, 9.0]), pos, vel, pbf, pbx, g, 2, seed)
    assert (g, imp) == (0, 1)
