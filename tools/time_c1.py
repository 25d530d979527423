"""C1 latency (32x32 single slice, C = 3, lambda = xi = 0.5, 20
IFCM iterations): device time per iteration of pifcm_iterate, CUDA events on
the launch stream.  Never a bench value.

    python tools/time_c1.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from inputs import CONFIGS, config_volume
from paper_2002_01981_b200 import Context, IfcmConfig, to_aos, to_pitched_x

ctx = Context(0)
cfgd = CONFIGS["C1"]
vol, _ = config_volume("C1")
C = cfgd["C"]
dev = torch.device("cuda:0")
vt = torch.as_tensor(vol, device=dev)
x, hist = ctx.normalize(vt)
nz, ny, nx = vol.shape
U = torch.full((1, nz * ny * nx, 4), 0.0, device=dev)
U[..., :C] = 1.0 / C
Un = torch.empty_like(U)
cen = torch.zeros((1, 4), device=dev)
cen[0, :C] = torch.tensor([0.1, 0.5, 0.9])
lx = torch.tensor([[cfgd["lam"], cfgd["xi"]]], dtype=torch.float64, device=dev)
cfg = IfcmConfig(C=C, eps=0.0)
out = {}
for iters in (1, 20):
    for _ in range(3):
        ctx.iterate(x, U, Un, cen, lx, cfg, iters=iters, nx=nx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        ctx.iterate(x, U, Un, cen, lx, cfg, iters=iters, nx=nx)
    e1.record()
    torch.cuda.synchronize()
    out[f"iters_{iters}"] = {"us_per_iteration": e0.elapsed_time(e1) * 1e3 / (reps * iters)}
out["workload"] = "C1: 32x32x1, C=3, lambda = xi = 0.5, P = 1 (pifcm_iterate)"
print(json.dumps(out, indent=1))
