"""Wall time of pifcm_segment on C3 (P = 32, 30 generations) for the three
fitness modes (CUDA events inside the library's report; never a bench value).

    python tools/time_modes.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import config_volume
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig

ctx = Context(0)
vol, _ = config_volume("C3")
nz, ny, nx = vol.shape
vt = torch.as_tensor(vol, device="cuda:0")
cfg = IfcmConfig(C=4)
out = {}
for mode, name in ((0, "chained"), (1, "anchored"), (2, "leader")):
    pso = PsoConfig(P=32, max_gen=30, patience=0, seed=12345, fitness=mode)
    ws = ctx.workspace(nx, ny, nz, cfg, pso)
    for _ in range(2):
        ctx.segment(vt, cfg, pso, ws=ws)
    reps = [ctx.segment(vt, cfg, pso, ws=ws)[2] for _ in range(3)]
    t_pso = sorted(r["t_pso"] for r in reps)[1]
    t_tot = sorted(r["t_total"] for r in reps)[1]
    out[name] = {"t_pso_ms": t_pso * 1e3, "t_total_ms": t_tot * 1e3, "ms_per_generation": t_pso * 1e3 / 30,
                 "lambda": reps[-1]["lambda"], "xi": reps[-1]["xi"], "workspace_GB": ws.numel() / 1e9}
    del ws
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
