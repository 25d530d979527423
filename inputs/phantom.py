"""Synthetic, seeded inputs with the shapes of the paper's workloads.

* ``cube_phantom``: the "cube within a cube with ranging grayscale colors"
  (§6.2.2), nested centred boxes; 2D when nz == 1 (the
  32x32 ... 854x854 images of Table 7).
* ``brainweb_phantom``: a BrainWeb-shaped 181x217x181 volume
  with BG / CSF / GM / WM as nested ellipsoids plus two CSF ventricles
  (reading R18 in DESIGN.md; the real BrainWeb data is out of scope).
* ``add_noise_u8``: additive iid Gaussian noise, sigma = pct/100 on the [0,1]
  scale, clamped, quantised to u8 (R17; "3% to 9%").
* ``random_state``: random membership rows / centres for parity tests.

No arithmetic of the 3DPIFCM method lives here.
"""
from __future__ import annotations

import numpy as np

__all__ = ["cube_phantom", "brainweb_phantom", "add_noise_u8", "random_state", "rng",
           "config_volume", "CONFIGS"]

LEVELS_C3 = (0.1, 0.5, 0.9)
LEVELS_C4 = (0.1, 0.35, 0.65, 0.9)
BRAINWEB_LEVELS = (0.0, 0.25, 0.55, 0.8)  # BG, CSF, GM, WM


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(int(seed)))


def cube_phantom(nx: int, ny: int, nz: int, levels=LEVELS_C4):
    """Nested centred boxes.  Region k (0 = outermost) holds the voxels whose
    per-axis normalised Chebyshev distance to the centre is <= 1 - k/R.
    Returns (clean float image in [0,1] [nz,ny,nx], truth labels u8)."""
    R = len(levels)
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    d = np.maximum(np.abs(xx + 0.5 - nx / 2) / (nx / 2), np.abs(yy + 0.5 - ny / 2) / (ny / 2))
    if nz > 1:
        d = np.maximum(d, np.abs(zz + 0.5 - nz / 2) / (nz / 2))
    lab = np.zeros((nz, ny, nx), np.uint8)
    for k in range(1, R):
        lab[d <= 1.0 - k / R] = k
    img = np.asarray(levels, np.float64)[lab]
    return img, lab


def brainweb_phantom(nx: int = 181, ny: int = 217, nz: int = 181):
    """BrainWeb-shaped head: BG(0), CSF(1), GM(2), WM(3) as nested ellipsoids
    with two CSF ventricles inside the WM.  Returns (clean image, labels)."""
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    u = (xx + 0.5 - nx / 2) / (nx / 2)
    v = (yy + 0.5 - ny / 2) / (ny / 2)
    w = (zz + 0.5 - nz / 2) / (nz / 2)
    # a slightly irregular radius so that tissue boundaries are not pure ellipsoids
    r = np.sqrt(u * u + v * v + w * w) * (1.0 + 0.04 * np.sin(5 * np.arctan2(v, u)) * np.cos(3 * w))
    lab = np.zeros((nz, ny, nx), np.uint8)
    lab[r <= 0.92] = 1
    lab[r <= 0.82] = 2
    lab[r <= 0.66] = 3
    for sx in (-1.0, 1.0):
        vent = ((u - 0.18 * sx) / 0.11) ** 2 + ((v - 0.05) / 0.28) ** 2 + (w / 0.16) ** 2 <= 1.0
        lab[vent] = 1
    img = np.asarray(BRAINWEB_LEVELS, np.float64)[lab]
    return img, lab


def add_noise_u8(img: np.ndarray, pct: float, seed: int) -> np.ndarray:
    """img in [0,1] + N(0, (pct/100)^2), clamped to [0,1], quantised to u8."""
    if pct < 0:
        raise ValueError("noise percentage must be >= 0")
    g = rng(seed)
    noisy = img + g.standard_normal(img.shape) * (pct / 100.0)
    return np.clip(np.rint(np.clip(noisy, 0.0, 1.0) * 255.0), 0, 255).astype(np.uint8)


def random_state(nx: int, ny: int, nz: int, C: int, seed: int, u8_levels: bool = True,
                 crisp_frac: float = 0.0):
    """Random (x, U, c) for step-parity tests.  x takes u8-derived values
    k/255 (so the G == 0 test is decided identically in fp32 and fp64), rows
    of U are random points of the simplex (a fraction crisp), centres in
    (0, 1).  Arrays are fp32 values (the GPU's storage precision)."""
    g = rng(seed)
    if u8_levels:
        x = (g.integers(0, 256, size=(nz, ny, nx)).astype(np.float64) / 255.0)
    else:
        x = g.random((nz, ny, nx))
    x = x.astype(np.float32)
    U = g.random((nz * ny * nx, C)) + 1e-3
    if crisp_frac > 0:
        crisp = g.random(U.shape[0]) < crisp_frac
        hot = g.integers(0, C, size=U.shape[0])
        U[crisp] = 0.0
        U[crisp, hot[crisp]] = 1.0
    U = U / U.sum(axis=1, keepdims=True)
    U = U.astype(np.float32)
    c = np.sort(g.random(C) * 0.9 + 0.05).astype(np.float32)
    return x, U, c


# The BASELINE.json configs.
CONFIGS = {
    "C1": dict(kind="cube", shape=(1, 32, 32), C=3, noise=7.0, seed=1, P=1, iters=20,
               lam=0.5, xi=0.5),
    "C2": dict(kind="cube", shape=(1, 854, 854), C=4, noise=7.0, seed=2, P=20, gens=30),
    "C3": dict(kind="brainweb", shape=(181, 217, 181), C=4, noise=9.0, seed=3, P=32, gens=30),
    "C5": dict(kind="cube", shape=(512, 512, 512), C=4, noise=7.0, seed=5, P=64, gens=30),
    # C4: a batch of 16 BrainWeb-shaped volumes, seeds 100..115, noise cycling
    # 3/5/7/9 %; volume k is config_volume("C4", k=k)
    "C4": dict(kind="brainweb", shape=(181, 217, 181), C=4, noise=(3.0, 5.0, 7.0, 9.0), seed=100, P=32,
               gens=30, batch=16),
}


def config_volume(name: str, shape=None, k: int = 0):
    """u8 noisy volume and truth labels for a named config (optionally
    reshaped); k selects the volume of a batch config (C4)."""
    cfg = CONFIGS[name]
    nz, ny, nx = shape if shape is not None else cfg["shape"]
    if cfg["kind"] == "cube":
        img, lab = cube_phantom(nx, ny, nz, LEVELS_C3 if cfg["C"] == 3 else LEVELS_C4)
    else:
        img, lab = brainweb_phantom(nx, ny, nz)
    noise = cfg["noise"]
    if isinstance(noise, tuple):
        noise = noise[k % len(noise)]
    return add_noise_u8(img, noise, cfg["seed"] + k), lab
