"""The seeded input generators (no method arithmetic)."""
import numpy as np

from inputs import add_noise_u8, brainweb_phantom, config_volume, cube_phantom, random_state


def test_cube_phantom_levels():
    img, lab = cube_phantom(32, 32, 1)
    assert set(np.unique(img).tolist()) == {0.1, 0.35, 0.65, 0.9}
    assert set(np.unique(lab).tolist()) == {0, 1, 2, 3}
    assert (img == img[:, ::-1, ::-1]).all()  # symmetric about the centre


def test_brainweb_shape():
    img, lab = brainweb_phantom(45, 54, 45)
    assert img.shape == (45, 54, 45)
    assert set(np.unique(lab).tolist()) == {0, 1, 2, 3}


def test_noise():
    img = np.full((64, 64, 16), 0.5)
    v0 = add_noise_u8(img, 0.0, 1)
    assert (v0 == 128).all()
    v = add_noise_u8(img, 5.0, 1).astype(np.float64) / 255.0
    assert abs((v - 0.5).std() - 0.05) < 0.0025
    assert (add_noise_u8(img, 5.0, 1) == add_noise_u8(img, 5.0, 1)).all()


def test_random_state():
    x, U, c = random_state(5, 4, 3, 4, 0, crisp_frac=0.3)
    assert x.dtype == np.float32 and U.shape == (60, 4)
    assert np.allclose(U.sum(1), 1, atol=1e-6)
    assert ((x * 255).round() == x * 255).all() or np.allclose((x * 255).round(), x * 255, atol=1e-4)


def test_config_volume_small():
    vol, lab = config_volume("C3", shape=(18, 22, 18))
    assert vol.dtype == np.uint8 and vol.shape == (18, 22, 18)
