"""Pins of the oracle's PSO (Alg. 1 steps 3-9), Philox, GMM init
and pipeline plumbing.  CPU only."""
import numpy as np
import pytest


def test_philox_known_answers(orc):
    """Random123 philox4x32-10 known-answer vectors (kat_vectors)."""
    assert [hex(v) for v in orc.philox4x32_10([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(v) for v in orc.philox4x32_10([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(v) for v in orc.philox4x32_10(
        [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])] == \
        ["0xd16cfe09", "0x94fdcceb", "0x5001e420", "0x24126ea1"]


def test_philox_u01(orc):
    """53-bit doubles from two words (R12): words (w0, w1) -> ((w1<<32|w0)>>11) 2^-53."""
    o = orc.philox4x32_10([7, 3, 0, 0], [12345, 0])
    a, b = orc.philox_pair(12345, 7, 3, 0, 0)
    assert a == float(((int(o[1]) << 32 | int(o[0])) >> 11)) / 2.0 ** 53
    assert b == float(((int(o[3]) << 32 | int(o[2])) >> 11)) / 2.0 ** 53
    draws = np.array([orc.philox_pair(99, g, p, 0, 0) for g in range(40) for p in range(50)])
    assert (draws >= 0).all() and (draws < 1).all()
    assert abs(draws.mean() - 0.5) < 0.02


def test_velocity_worked_example(orc):
    """SPEC:376 on Alg. 1 step 7: v=0, pbest-x=(0.2,0), lbest-x=(0,0.2), p1=p2=1 -> (0.2,0.2)."""
    pos = np.array([[0.3, 0.3], [0.3, 0.5]])
    vel = np.zeros((2, 2))
    pbest_x = np.array([[0.5, 0.3], [0.3, 0.5]])
    orc.pso_move(pos, vel, pbest_x, [1, 1], [1.0, 1.0], [1.0, 1.0])
    assert np.allclose(vel[0], [0.2, 0.2], atol=1e-15)
    assert np.allclose(pos[0], [0.5, 0.5], atol=1e-15)
    # clamp: |v| <= 0.5 and x in [0,1]
    pos = np.array([[0.9, 0.1]])
    vel = np.array([[0.45, -0.45]])
    orc.pso_move(pos, vel, np.array([[1.9, -0.9]]), [0], [1.0], [0.0])
    assert vel.tolist() == [[0.5, -0.5]] and pos.tolist() == [[1.0, 0.0]]


def test_velocity_fixed_point(orc):
    """x = pbest = lbest -> velocity unchanged."""
    pos = np.array([[0.4, 0.6]])
    vel = np.array([[0.01, -0.02]])
    orc.pso_move(pos, vel, pos.copy(), [0], [0.7], [0.3])
    assert np.allclose(vel, [[0.01, -0.02]])


def _run_pso(orc, fit, P=10, gens=60, seed=5):
    pos, vel = orc.pso_init(P, seed)
    pbf = np.full(P, np.inf)
    pbx = pos.copy()
    g = -1
    hist = []
    for t in range(gens):
        f = np.array([fit(p) for p in pos])
        g, _ = orc.pso_update(f, pos, vel, pbf, pbx, g, t, seed)
        hist.append(pbf[g])
        assert (pos >= 0).all() and (pos <= 1).all()
    return np.array(hist), pbf, pbx, g


def test_pso_quadratic(orc):
    """f = lambda^2 + xi^2 -> best < 0.01; gbest monotone."""
    hist, pbf, pbx, g = _run_pso(orc, lambda p: p[0] ** 2 + p[1] ** 2)
    assert hist[-1] < 0.01
    assert (np.diff(hist) <= 0).all()


def test_pso_constant_fitness(orc):
    """Constant fitness -> pbest positions never change after the first evaluation."""
    P, seed = 6, 3
    pos, vel = orc.pso_init(P, seed)
    pbf = np.full(P, np.inf)
    pbx = pos.copy()
    g = -1
    g, imp = orc.pso_update(np.ones(P), pos, vel, pbf, pbx, g, 0, seed)
    assert imp == 1 and g == 0  # ties -> lowest index
    first = pbx.copy()
    for t in range(1, 10):
        g, imp = orc.pso_update(np.ones(P), pos, vel, pbf, pbx, g, t, seed)
        assert imp == 0 and g == 0
    assert (pbx == first).all()


def test_pso_single_particle(orc):
    """P = 1: the ring is {0}, lbest == pbest."""
    pos, vel = orc.pso_init(1, 8)
    pbf = np.full(1, np.inf)
    pbx = pos.copy()
    g, imp = orc.pso_update(np.array([2.0]), pos, vel, pbf, pbx, -1, 0, 8)
    assert g == 0 and imp == 1


def test_pso_init_ranges(orc):
    pos, vel = orc.pso_init(64, 42, v0=0.1)
    assert (pos >= 0).all() and (pos < 1).all()
    assert (np.abs(vel) <= 0.1).all()
    pos2, vel2 = orc.pso_init(64, 42, v0=0.1)
    assert (pos == pos2).all() and (vel == vel2).all()


def test_pso_run_on_step_fitness(orc):
    """CHAINED PSO on a tiny noisy phantom: gbest monotone, positions in range,
    J at (lambda*, xi*) <= J at (0, 0) from the same state."""
    from inputs import cube_phantom, add_noise_u8
    img, _ = cube_phantom(10, 10, 3, (0.1, 0.5, 0.9))
    x = add_noise_u8(img, 7.0, 4).astype(np.float64) / 255.0
    U0, c0, _ = orc.fcm_run(x, np.array([0.1, 0.5, 0.9]))
    r = orc.pso_run(x, U0, c0, P=6, max_gen=8, seed=77)
    assert r.generations == 8
    gb = np.minimum.accumulate(r.trace_f.min(1))
    assert abs(gb[-1] - r.J) < 1e-15
    assert (r.trace_pos >= 0).all() and (r.trace_pos <= 1).all()
    _, _, J00, _ = orc.ifcm_step(x, U0, c0, 0.0, 0.0)
    assert r.trace_f[0].min() <= J00 + 1e-15


def _mode_problem(orc):
    from inputs import add_noise_u8, cube_phantom
    img, _ = cube_phantom(10, 9, 3, (0.1, 0.5, 0.9))
    x = add_noise_u8(img, 7.0, 4).astype(np.float64) / 255.0
    U0, c0, _ = orc.fcm_run(x, np.array([0.1, 0.5, 0.9]))
    return x, U0, c0


def _assert_monotone(pos, f):
    """From one fixed state J is non-increasing in lambda and in xi (pinned in
    test_oracle_pins.test_cost_monotone_in_lambda_xi): any two evaluations of
    the same state must be ordered accordingly."""
    for a in range(len(f)):
        for b in range(len(f)):
            if pos[a, 0] <= pos[b, 0] and pos[a, 1] <= pos[b, 1]:
                assert f[a] >= f[b] - 1e-12 * abs(f[b]), (pos[a], pos[b], f[a], f[b])


def test_pso_anchored_mode(orc):
    """ANCHORED: every evaluation is one step from the
    shared start, so (i) every fitness of the run is ordered by the
    monotonicity of J in (lambda, xi) -- across all generations --, (ii) the
    first generation equals CHAINED's, (iii) the gbest snapshot is the step
    from the start at (lambda*, xi*)."""
    x, U0, c0 = _mode_problem(orc)
    r = orc.pso_run(x, U0, c0, P=6, max_gen=6, seed=77, fitness_mode=1)
    rc = orc.pso_run(x, U0, c0, P=6, max_gen=1, seed=77, fitness_mode=0)
    assert (r.trace_f[0] == rc.trace_f[0]).all()
    _assert_monotone(r.trace_pos.reshape(-1, 2), r.trace_f.ravel())
    Ub, cb, Jb, _ = orc.ifcm_step(x, U0, c0, r.lam, r.xi)
    assert Jb == r.J and (Ub == r.U).all() and (cb == r.c).all()
    assert r.J == r.trace_f.min()


def test_pso_leader_mode(orc):
    """LEADER (R22): within a generation all evaluations share one state
    (monotonicity per generation); generation 0 equals ANCHORED's; generation
    1 is evaluated from the state the gbest's generation-0 evaluation produced."""
    x, U0, c0 = _mode_problem(orc)
    r = orc.pso_run(x, U0, c0, P=5, max_gen=4, seed=91, fitness_mode=2)
    ra = orc.pso_run(x, U0, c0, P=5, max_gen=1, seed=91, fitness_mode=1)
    assert (r.trace_f[0] == ra.trace_f[0]).all()
    for g in range(4):
        _assert_monotone(r.trace_pos[g], r.trace_f[g])
    g0 = r.trace_gbest[0]
    U1, c1, _, _ = orc.ifcm_step(x, U0, c0, *r.trace_pos[0, g0])
    for p in range(5):
        _, _, J, _ = orc.ifcm_step(x, U1, c1, *r.trace_pos[1, p])
        assert J == r.trace_f[1, p]


def test_pso_early_stop(orc):
    from inputs import cube_phantom
    img, _ = cube_phantom(8, 8, 2, (0.1, 0.9))
    U0, c0, _ = orc.fcm_run(img, np.array([0.2, 0.8]))
    r = orc.pso_run(img, U0, c0, P=4, max_gen=30, seed=1, patience=3, tol=1e-4)
    assert r.generations < 30


# --------------------------------------------------------------------------- GMM init (R15)
def test_gmm_two_modes(orc):
    """EM on a two-intensity histogram converges to the modes."""
    h = np.zeros(256, np.int64)
    h[51] = 500   # 0.2
    h[204] = 700  # 0.8
    c = orc.gmm_init(h, 2)
    assert np.allclose(c, [51 / 255, 204 / 255], atol=1e-6)


def test_gmm_fallback_and_determinism(orc):
    h = np.zeros(256, np.int64)
    h[100] = 10
    assert np.allclose(orc.gmm_init(h, 3), [0.0, 0.5, 1.0])
    rng = np.random.default_rng(3)
    h = rng.integers(0, 100, 256)
    assert (orc.gmm_init(h, 4) == orc.gmm_init(h, 4)).all()
    c = orc.gmm_init(h, 4)
    assert (np.diff(c) > 0).all() and (c >= 0).all() and (c <= 1).all()


def test_gmm_phantom_levels(orc):
    """Noisy 4-level phantom: the GMM means land near the true levels."""
    from inputs import cube_phantom, add_noise_u8
    img, _ = cube_phantom(48, 48, 8)
    vol = add_noise_u8(img, 3.0, 1)
    c = orc.gmm_init(orc.histogram_u8(vol), 4)
    assert np.allclose(c, [0.1, 0.35, 0.65, 0.9], atol=0.03)


def test_fcm_run_converges(orc):
    from inputs import cube_phantom, add_noise_u8
    img, lab = cube_phantom(20, 20, 1, (0.1, 0.5, 0.9))
    x = add_noise_u8(img, 5.0, 2).astype(np.float64) / 255.0
    U, c, t = orc.fcm_run(x, np.array([0.0, 0.4, 1.0]), eps=1e-5)
    assert t < 100
    assert np.allclose(np.sort(c), [0.1, 0.5, 0.9], atol=0.03)


def test_segment_small(orc):
    """Pipeline plumbing on a small noisy phantom.  Under J-fitness the swarm is
    driven towards lambda = xi = 1 (J is non-increasing in both, see
    test_cost_monotone_in_lambda_xi), so no interior optimum or label quality
    is asserted; only ranges and that the gbest J beats the FCM point."""
    from inputs import cube_phantom, add_noise_u8
    img, lab = cube_phantom(16, 16, 6, (0.1, 0.5, 0.9))
    vol = add_noise_u8(img, 7.0, 3)
    r = orc.segment_u8(vol, C=3, P=4, max_gen=4, seed=5)
    assert r.labels.shape == vol.shape and r.labels.max() <= 2
    assert 0 <= r.lam <= 1 and 0 <= r.xi <= 1
    assert r.generations == 4 and 1 <= r.final_iters <= 100
    x = orc.normalize_u8(vol)
    U, c, _ = orc.fcm_run(x, r.c_init)
    _, _, J00, _ = orc.ifcm_step(x, U, c, 0.0, 0.0)
    assert r.J <= J00
    assert (np.diff(np.sort(r.c)) > 0).all()


def test_segment_equals_its_parts(orc):
    """orc_segment_u8 = gmm_init -> fcm_run -> pso_run -> ifcm_run -> argmax
    (Alg. 1 steps 2-11): the end-to-end GPU test at C3 runs the
    oracle through these parts to get the swarm trace, so they must compose to
    the whole pipeline exactly."""
    from inputs import add_noise_u8, cube_phantom
    img, _ = cube_phantom(20, 18, 6, (0.1, 0.35, 0.65, 0.9))
    vol = add_noise_u8(img, 9.0, 11)
    r = orc.segment_u8(vol, C=4, P=5, max_gen=4, seed=99)
    x = orc.normalize_u8(vol)
    c0 = orc.gmm_init(orc.histogram_u8(vol), 4)
    U1, c1, _ = orc.fcm_run(x, c0)
    p = orc.pso_run(x, U1, c1, P=5, max_gen=4, seed=99)
    Uf, cf, it, _ = orc.ifcm_run(x, p.U, p.c, p.lam, p.xi)
    assert (p.lam, p.xi) == (r.lam, r.xi)
    assert it == r.final_iters
    assert np.array_equal(orc.argmax(Uf).reshape(vol.shape), r.labels)
    assert np.array_equal(cf, r.c)
