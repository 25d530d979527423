"""Multi-GPU readiness on one GPU (Sec. 7 names the
single GPU as the paper's limitation): bench.py launched as the driver
launches it for N = 2 (torchrun, one process per rank, 127.0.0.1
rendezvous), with the gloo backend so the two ranks can share the one B200
of this box.  The N = 2 line must keep the JSON contract and the particle-
sharded pipeline must reproduce the N = 1 segmentation bit for bit (labels,
lambda*, xi*, final iterations): the fitness all-gather and the gbest
broadcast change nothing in the arithmetic."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(cmd, dump, extra_env):
    env = dict(os.environ, PIFCM_BENCH_DUMP=dump, **extra_env)
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_bench_two_ranks_match_one(tmp_path):
    base = [sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    one = _run(base, str(tmp_path / "n1.npz"), {})
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
                "--steps", "1", "--warmup", "3", "--no-cpu-baseline"],
               str(tmp_path / "n2.npz"), {"PIFCM_BENCH_BACKEND": "gloo"})
    for line, n in ((one, 1), (two, 2)):
        assert KEYS <= set(line), KEYS - set(line)
        assert line["n_gpus"] == n and line["steps"] == 1 and line["warmup"] == 3
        assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
        assert line["config"]["workload"].startswith("C3")
    assert two["config"]["parallelism"].startswith("particles/2")
    a, b = np.load(tmp_path / "n1.npz"), np.load(tmp_path / "n2.npz")
    assert np.array_equal(a["lam_xi"], b["lam_xi"])
    assert int(a["final_iters"]) == int(b["final_iters"])
    assert np.array_equal(a["labels"], b["labels"])
