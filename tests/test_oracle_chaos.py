"""The reading DESIGN.md §7 gives for the end-to-end fitness comparison: with
J-fitness the swarm drives every particle to lambda = xi = 1 (Eq. 4
with the floor R4), where the chained IFCM map (Alg. 1 steps 4-10,
PAPER:98-104) amplifies rounding-level differences of a particle's state.
Pinned here on the oracle alone (no GPU): the same swarm run twice, once from
the fp64 FCM start and once from that start rounded to fp32 -- the precision
the GPU path stores -- must agree at first to the rounding level and then
drift apart by orders of magnitude, while the positions (fp64 PSO arithmetic
deciding on pbest comparisons) stay bit-identical.  This is why the C3
end-to-end test (tests/test_gpu_c3_e2e.py) asserts fitness within 1e-5 only
for the first generations and compares deep generations from the same state."""
import numpy as np


def test_fp32_rounding_of_the_start_grows_along_the_swarm(orc):
    from inputs import add_noise_u8, brainweb_phantom
    img, _ = brainweb_phantom(40, 48, 40)
    vol = add_noise_u8(img, 9.0, 3)
    x = orc.normalize_u8(vol)
    c0 = orc.gmm_init(orc.histogram_u8(vol), 4)
    U1, c1, _ = orc.fcm_run(x, c0)
    G = 30
    a = orc.pso_run(x, U1, c1, P=32, max_gen=G, seed=12345)
    r32 = lambda v: np.asarray(v).astype(np.float32).astype(np.float64)  # noqa: E731
    b = orc.pso_run(r32(x), r32(U1), r32(c1), P=32, max_gen=G, seed=12345)
    rel = np.abs(a.trace_f - b.trace_f) / np.abs(a.trace_f)
    # the trajectory is decided by comparisons only: identical positions
    assert np.array_equal(a.trace_pos, b.trace_pos)
    assert (a.lam, a.xi) == (b.lam, b.xi) == (1.0, 1.0)
    # the first generations agree to the rounding level ...
    assert rel[:5].max() < 1e-6, rel[:5].max(axis=1)
    # ... and the difference grows by orders of magnitude along the swarm
    assert rel[-5:].max() > 1e-3, rel.max(axis=1)
    assert rel[-5:].max() > 1e3 * rel[0].max()
