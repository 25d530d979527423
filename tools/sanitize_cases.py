"""Small cases for compute-sanitizer (tools/sanitize.sh): every device kernel
of the hot path once, through the C ABI, on inputs small enough that the
sanitizer's instrumentation finishes in seconds.

    python tools/sanitize_cases.py [case ...]

Cases: c1 (32x32 image, 20 iterations: the one-launch small-2D kernel),
3d (12x12x5 and a 19x37x70 multi-tile volume, P = 3: the TMA-ring stencil
kernel with the fp64 band pass), 2d (96x97 and 140x41 images: k_step_2d),
v2 (two-shell kernel), pipe (pifcm_segment on a small phantom: normalise,
histograms, GMM, FCM start, PSO, final IFCM, argmax), modes (ANCHORED /
LEADER fitness), slab (a two-slab split of the final IFCM through the
z-slab ABI).  The PSO thread-contention hazard the paper names (PAPER:122,
Sec. 3) lives in the ring refill and the last-CTA finalisation, which every
case exercises."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import add_noise_u8, cube_phantom, random_state  # noqa: E402
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig, to_aos, to_pitched_x  # noqa: E402

DEV = torch.device("cuda:0")


def _iterate(ctx, shape, C, P, iters, lam=(0.9, 1.0), v=1, m=2.0, canonical=False):
    nz, ny, nx = shape
    xs, Us, cs = [], [], []
    for p in range(P):
        x, U, c = random_state(nx, ny, nz, C, seed=10 + p, crisp_frac=0.1)
        Us.append(U)
        cs.append(c)
    xt = to_pitched_x(x, DEV)
    Uin = to_aos(np.stack(Us), DEV)
    Uout = torch.empty_like(Uin)
    cen = torch.zeros((P, 4), device=DEV)
    cen[:, :C] = torch.as_tensor(np.stack(cs), dtype=torch.float32)
    lx = torch.tensor([lam] * P, dtype=torch.float64, device=DEV)
    stats = torch.zeros((P, 4), dtype=torch.float64, device=DEV)
    ctx.iterate(xt, Uin, Uout, cen, lx, IfcmConfig(C=C, v=v, m=m, eps=1e-5), iters=iters, stats=stats, nx=nx,
                canonical=canonical)
    torch.cuda.synchronize()
    assert torch.isfinite(Uout).all()


def case_c1(ctx):
    _iterate(ctx, (1, 32, 32), 3, 1, 20, lam=(0.5, 0.5))


def case_3d(ctx):
    _iterate(ctx, (5, 12, 12), 4, 1, 2)
    _iterate(ctx, (19, 37, 70), 4, 3, 2, lam=(1.0, 1.0))
    _iterate(ctx, (9, 17, 33), 3, 2, 1, m=1.5)
    _iterate(ctx, (19, 37, 70), 4, 1, 2, canonical=True)


def case_2d(ctx):
    _iterate(ctx, (1, 96, 97), 4, 2, 2)
    _iterate(ctx, (1, 140, 41), 3, 1, 2, m=1.5)


def case_v2(ctx):
    _iterate(ctx, (9, 17, 33), 4, 2, 1, v=2)


def _phantom():
    img, _ = cube_phantom(24, 20, 8, (0.1, 0.5, 0.9))
    return add_noise_u8(img, 7.0, 3)


def case_pipe(ctx):
    vol = torch.as_tensor(_phantom(), device=DEV)
    labels, _, rep = ctx.segment(vol, IfcmConfig(C=3), PsoConfig(P=4, max_gen=3, patience=0, seed=7))
    torch.cuda.synchronize()
    assert int(labels.max()) <= 2


def case_modes(ctx):
    vol = torch.as_tensor(_phantom(), device=DEV)
    for mode in (1, 2):
        ctx.segment(vol, IfcmConfig(C=3), PsoConfig(P=4, max_gen=2, patience=0, seed=7, fitness=mode))
    torch.cuda.synchronize()


def case_slab(ctx):
    from paper_2002_01981_b200.dist import SlabIfcm
    nx, ny, nz, C, P = 37, 30, 40, 4, 1
    x, U, c = random_state(nx, ny, nz, C, seed=61, crisp_frac=0.1)

    s = SlabIfcm(ctx, IfcmConfig(C=C), nx, ny, nz, P, None)
    s.load_x(to_pitched_x(x, DEV))
    cen = torch.zeros((P, 4), device=DEV)
    cen[:, :C] = torch.as_tensor(c)
    s.load_state(to_aos(U[None], DEV).view(1, -1, 4), cen)
    s.run(torch.tensor([[0.6, 0.8]], dtype=torch.float64, device=DEV), 3, eps=0.0)
    torch.cuda.synchronize()


CASES = {"c1": case_c1, "3d": case_3d, "2d": case_2d, "v2": case_v2, "pipe": case_pipe, "modes": case_modes,
         "slab": case_slab}


def main(argv):
    names = argv or list(CASES)
    ctx = Context(0)
    for n in names:
        CASES[n](ctx)
        print(f"case {n} ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
