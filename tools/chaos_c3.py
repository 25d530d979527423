"""The oracle against itself at the bench configuration (C3, P = 32, 30
generations, seed 12345): the whole pipeline once from the fp64 FCM start and
once from that start rounded to fp32 (the GPU path's storage precision).  The
per-generation fitness differences between the two are the yardstick for the
GPU-vs-oracle differences recorded by tests/test_gpu_c3_e2e.py.
CPU only (~20 min on 16 host cores).

    python tools/chaos_c3.py gpurun_out/chaos_c3.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc  # noqa: E402
from inputs import config_volume  # noqa: E402

P, G, SEED, C = 32, 30, 12345, 4
vol, _ = config_volume("C3")
x = orc.normalize_u8(vol)
c0 = orc.gmm_init(orc.histogram_u8(vol), C)
U1, c1, _ = orc.fcm_run(x, c0)
r32 = lambda v: np.asarray(v).astype(np.float32).astype(np.float64)  # noqa: E731
t0 = time.time()
runs = []
for xs, Us, cs in ((x, U1, c1), (r32(x), r32(U1), r32(c1))):
    r = orc.pso_run(xs, Us, cs, P=P, max_gen=G, seed=SEED)
    Uf, cf, it, _ = orc.ifcm_run(xs, r.U, r.c, r.lam, r.xi)
    runs.append((r, orc.argmax(Uf), it, cf))
(a, la, ia, ca), (b, lb, ib, cb) = runs
rel = np.abs(a.trace_f - b.trace_f) / np.abs(a.trace_f)
out = {
    "what": "oracle vs oracle from the fp32-rounded FCM start, C3 bench configuration",
    "host_threads": orc.num_threads(), "seconds": time.time() - t0,
    "fitness_max_rel_by_generation": rel.max(axis=1).tolist(),
    "fitness_median_rel_by_generation": np.median(rel, axis=1).tolist(),
    "positions_identical": bool(np.array_equal(a.trace_pos, b.trace_pos)),
    "gbest_identical": bool(np.array_equal(a.trace_gbest, b.trace_gbest)),
    "lambda_xi": [[a.lam, a.xi], [b.lam, b.xi]], "final_iters": [ia, ib],
    "centers": [ca.tolist(), cb.tolist()],
    "label_agreement": float((la == lb).mean()),
}
with open(sys.argv[1] if len(sys.argv) > 1 else "chaos_c3.json", "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))
