"""Device time of the fused step for v = 1, 2 and 3 (NEXT-2) on C3, P = 32
(one PSO generation per launch; CUDA events on the launch stream via the
library's timing; never a bench value).

    python tools/time_shells.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import config_volume
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
from paper_2002_01981_b200.api import _grid

ctx = Context(0)
vol, _ = config_volume("C3")
nz, ny, nx = vol.shape
vt = torch.as_tensor(vol, device="cuda:0")
out = {}
for v in (1, 2, 3):
    cfg = IfcmConfig(C=4, v=v, h=1.0)
    pso = PsoConfig(P=32, max_gen=30, patience=0, seed=12345)
    ws = ctx.workspace(nx, ny, nz, cfg, pso)
    x, hist = ctx.normalize_u8(vt)
    c0 = ctx.gmm_init(hist, 4)
    U0 = torch.full((nz * ny * nx, 4), 0.25, device="cuda:0")
    g = _grid(nx, ny, nz)
    ctx.pso_init(g, cfg, pso, U0, c0, ws)
    for _ in range(2):
        ctx.pso_step(g, cfg, pso, x, ws)
    ctx.timing_enable(True)
    for _ in range(6 if v < 3 else 2):
        ctx.pso_step(g, cfg, pso, x, ws)
    ms, n, b = ctx.timing_read()
    ctx.timing_enable(False)
    out[f"v{v}"] = {"ms_per_launch": ms / n, "G_vp_per_s": 32 * nz * ny * nx / (ms / n * 1e-3) / 1e9,
                    "neighbours": (2 * v + 1) ** 3 - 1}
    del ws
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
