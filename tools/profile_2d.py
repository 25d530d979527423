"""Workload for an ncu capture of the 2D step (C2, P = 20); never a bench number."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import config_volume
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
from paper_2002_01981_b200.api import _grid

ctx = Context(0)
vol, _ = config_volume("C2")
nz, ny, nx = vol.shape
cfg = IfcmConfig(C=4)
pso = PsoConfig(P=20, max_gen=30, patience=0, seed=12345)
ws = ctx.workspace(nx, ny, nz, cfg, pso)
vt = torch.as_tensor(vol, device="cuda:0")
x, hist = ctx.normalize_u8(vt)
c0 = ctx.gmm_init(hist, 4)
U0 = torch.full((nz * ny * nx, 4), 0.25, device="cuda:0")
g = _grid(nx, ny, nz)
ctx.pso_init(g, cfg, pso, U0, c0, ws)
for _ in range(3):
    ctx.pso_step(g, cfg, pso, x, ws)
torch.cuda.synchronize()
print("done")
