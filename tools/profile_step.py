"""Workloads for ncu captures (never a bench number).

  python tools/profile_step.py segment   # one whole C3 pifcm_segment (bench step)
  python tools/profile_step.py eval      # one generation of the fused step, P=32, C3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import config_volume
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
from paper_2002_01981_b200.api import _grid

mode = sys.argv[1] if len(sys.argv) > 1 else "segment"
# "time": device time per launch of the P = 32 fused step and of the
# single-state canonical launches of the final IFCM (CUDA events)
ctx = Context(0)
vol, _ = config_volume("C3")
nz, ny, nx = vol.shape
cfg = IfcmConfig(C=4)
pso = PsoConfig(P=32, max_gen=30, patience=0, seed=12345)
ws = ctx.workspace(nx, ny, nz, cfg, pso)
vt = torch.as_tensor(vol, device="cuda:0")
if mode == "segment":
    ctx.segment(vt, cfg, pso, ws=ws)
if mode in ("eval", "time"):
    x, hist = ctx.normalize_u8(vt)
    c0 = ctx.gmm_init(hist, 4)
    U0 = torch.full((nz * ny * nx, 4), 0.25, device="cuda:0")
    g = _grid(nx, ny, nz)
    ctx.pso_init(g, cfg, pso, U0, c0, ws)
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
        ctx.pso_step(g, cfg, pso, x, ws)
torch.cuda.synchronize()
print("done")

if mode == "time":
    # device time of the fused step at P=32 (C3), CUDA events on the launch stream
    ctx.timing_enable(True)
    for _ in range(10):
        ctx.pso_step(g, cfg, pso, x, ws)
    ms, n, b = ctx.timing_read()
    print(f"fused step: {ms / n:.3f} ms/launch, {b / n / 1e9:.3f} GB alg/launch, "
          f"{(b / n) / (ms / n * 1e-3) / 1e9:.1f} GB/s, {32 * nz * ny * nx / (ms / n * 1e-3) / 1e9:.1f} G vp/s")

if mode == "time":
    # single-state canonical launches (the final IFCM's decomposition)
    nvox = nz * ny * nx
    Ua = U0.view(1, nvox, 4).clone()
    Ub = torch.empty_like(Ua)
    cen = c0.clone().view(1, 4)
    lx = torch.tensor([[1.0, 1.0]], dtype=torch.float64, device="cuda:0")
    for _ in range(5):
        ctx.iterate(x, Ua, Ub, cen, lx, cfg, iters=1, nx=nx, canonical=True)
        Ua, Ub = Ub, Ua
    ctx.timing_enable(False)
    ctx.timing_enable(True)
    for _ in range(40):
        ctx.iterate(x, Ua, Ub, cen, lx, cfg, iters=1, nx=nx, canonical=True)
        Ua, Ub = Ub, Ua
    ms, n, b = ctx.timing_read(batched=False)
    print(f"single state: {ms / n * 1e3:.1f} us/launch, {(b / n) / (ms / n * 1e-3) / 1e9:.1f} GB/s")
