"""Label agreement GPU vs oracle for whole pipelines that end at
lambda* = xi* ~ 1 (the regime the small-case tests used to skip); prints one
JSON line per case.  Test aid, not a bench."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import oracle as orc
from inputs import add_noise_u8, cube_phantom
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig

ctx = Context(0)
cases = [
    # (C, shape (nz, ny, nx), P, G, seed, mode, v)
    (4, (12, 30, 33), 6, 4, 3, 1, 1), (4, (12, 30, 33), 6, 4, 3, 2, 1),
    (3, (10, 24, 28), 4, 8, 99, 0, 1), (4, (6, 33, 35), 5, 8, 1, 0, 1), (4, (1, 64, 64), 6, 8, 5, 0, 1),
    (4, (20, 40, 44), 8, 10, 7, 0, 1), (3, (10, 24, 28), 4, 8, 99, 0, 2),
]
for C, shape, P, G, seed, mode, v in cases:
    nz, ny, nx = shape
    img, _ = cube_phantom(nx, ny, nz, (0.1, 0.5, 0.9) if C == 3 else (0.1, 0.35, 0.65, 0.9))
    vol = add_noise_u8(img, 7.0, 11 if mode == 0 else 8)
    cfg = IfcmConfig(C=C, v=v)
    pso = PsoConfig(P=P, max_gen=G, patience=0, seed=seed, fitness=mode)
    lab, _, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), cfg, pso)
    r = orc.segment_u8(vol, C=C, P=P, max_gen=G, seed=seed, fitness_mode=mode, v=v)
    print(json.dumps({"case": [C, shape, P, G, seed, mode, v], "lam_xi_gpu": [rep["lambda"], rep["xi"]],
                      "lam_xi_orc": [r.lam, r.xi], "agree": float((lab.cpu().numpy() == r.labels).mean()),
                      "final_iters": [rep["final_iters"], r.final_iters],
                      "centers_maxrel": float(np.max(np.abs(np.array(rep["centers"]) - r.c) / np.abs(r.c)))}),
          flush=True)
