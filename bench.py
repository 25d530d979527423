#!/usr/bin/env python
"""Benchmark of the 3DPIFCM hot path on B200 (BASELINE.json metric:
"voxel-iterations/s (x particles) and PSO-3DPIFCM wall time, 181x217x181").

One step = one whole PSO-3DPIFCM segmentation (pifcm_segment: normalise ->
GMM -> FCM start -> 30 generations x 32 particles of the fused IFCM step ->
final IFCM until eps -> argmax) of the BrainWeb-shaped 181x217x181 synthetic
phantom (9% noise, C=4), early stop disabled so the work is fixed.
value = voxel x particle x iterations processed / second (all ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): particles are sharded over ranks (P/N each); the only
collectives are an all-gather of the per-particle fitness every generation and
a broadcast of the gbest state (paper_2002_01981_b200/dist.py).
--impl reference times the fp64 CPU oracle (the paper has no released code):
one step = one oracle IFCM step of one particle over the same volume.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "C3: BrainWeb-shaped 181x217x181 synthetic phantom (CSF/GM/WM), 9% noise, C=4, 26-neighbour 3D IFCM, PSO 32 particles x 30 generations"
WORKLOAD_C5 = ("C5: 512x512x512 synthetic noisy volume (4 nested cubes, 7% noise), C=4, z-slab sharded "
               "(halo exchange + record all-gather), PSO {P} particles x 30 generations")
WORKLOAD_C4 = ("C4: batch of 16 BrainWeb-shaped 181x217x181 volumes (seeds 100..115, noise 3/5/7/9%), C=4, "
               "26-neighbour 3D IFCM, PSO 32 particles x 30 generations each, particles sharded over the GPUs")
WORKLOAD_C2 = ("C2: 854x854 2D synthetic noisy image (4 nested squares, 7% noise), C=4, 8-neighbour IFCM, "
               "PSO 20 particles x 30 generations")
# PAPER:250 (Table 7, 3DPIFCM-GPU on a TITAN X, whole algorithm, 854x854): context only
PAPER_C2_SECONDS = 170.60
METRIC = "voxel-iterations/s (x particles)"
SHAPE = (181, 217, 181)  # (nz, ny, nx) with nx = 181, ny = 217, nz = 181
C, P, GENS = 4, 32, 30
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "kstep_summary.json")


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region: started
    before the warm-up (nvidia-smi needs ~0.1 s to its first sample), every
    sample time-stamped, only those inside [mark(), stop()] kept -- a timed
    region shorter than the sampling period keeps the sample nearest to it
    ("samples": 0)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        """The timed region starts now."""
        self.t0 = time.time()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        time.sleep(0.12)  # one more sample after the region, for the nearest-sample fallback
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [ln for t, ln in self.lines if t0 <= t <= t1]
        nearest = False
        if not inside and self.lines:
            mid = 0.5 * (t0 + t1)
            inside = [min(self.lines, key=lambda tl: abs(tl[0] - mid))[1]]
            nearest = True
        for ln in inside:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": 0 if nearest else len(sm)}


def _volume(name="C3"):
    from inputs import config_volume
    vol, _ = config_volume(name)
    return vol


def host_info(threads):
    """CPU model, logical CPUs and OMP_NUM_THREADS of the host the oracle ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except Exception:
        avail = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity_cpus": avail,
            "omp_num_threads_env": os.environ.get("OMP_NUM_THREADS"), "threads_used": threads}


def cpu_baseline_measure(vol, budget_s=20.0, P=P):
    """The oracle as it stands (fp64 C, OpenMP on all host cores) on a bounded
    sample of the same workload: whole IFCM steps of single particles over the
    full volume, repeated until ~budget_s of CPU work; plus one step on one
    thread (SURVEY 8(d)'s "sequential" point, in the spirit of Table 7's CPU
    column)."""
    import oracle
    x = oracle.normalize_u8(vol)
    c0 = oracle.gmm_init(oracle.histogram_u8(vol), C)
    U, c, _ = oracle.fcm_run(x, c0, max_iter=1)
    pos, _ = oracle.pso_init(P, 12345)
    n_vox = vol.size
    cores = oracle.num_threads()
    steps = 0
    t0 = time.perf_counter()
    while True:
        p = steps % P
        oracle.ifcm_step(x, U, c, pos[p, 0], pos[p, 1], m=2.0)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= 64:
            break
    seq = None
    try:
        oracle.set_num_threads(1)
        t1 = time.perf_counter()
        oracle.ifcm_step(x, U, c, pos[0, 0], pos[0, 1], m=2.0)
        e1 = time.perf_counter() - t1
        seq = {"value": n_vox / e1, "cores": 1, "sample": f"1 oracle IFCM step on one thread, {e1:.1f} s"}
    finally:
        oracle.set_num_threads(cores)
    return {"value": n_vox * steps / el, "unit": "voxel-iterations/s (x particles)",
            "cores": cores, "kind": "oracle", "host": host_info(cores),
            "sample": f"{steps} oracle IFCM steps (one particle each, lambda/xi from the bench "
                      f"swarm) over the full {'x'.join(map(str, vol.shape[::-1]))} volume, {el:.1f} s",
            "sequential": seq}


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle timed on host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    oracle.build_oracle()
    # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 runs the oracle
    # alone (the other ranks have exited), so it gets the host's cores
    try:
        oracle.set_num_threads(len(os.sched_getaffinity(0)))
    except Exception:
        pass
    c5 = args.workload == "C5"
    vol = _volume(args.workload)
    workload = (WORKLOAD_C5.format(P=64) if c5 else
                (WORKLOAD_C2 if args.workload == "C2" else WORKLOAD))
    x = oracle.normalize_u8(vol)
    c0 = oracle.gmm_init(oracle.histogram_u8(vol), C)
    U, c, _ = oracle.fcm_run(x, c0, max_iter=1)
    pos, _ = oracle.pso_init(P, 12345)
    for w in range(args.warmup):
        oracle.ifcm_step(x, U, c, pos[w % P, 0], pos[w % P, 1])
    t0 = time.perf_counter()
    for s in range(args.steps):
        oracle.ifcm_step(x, U, c, pos[s % P, 0], pos[s % P, 1])
    el = time.perf_counter() - t0
    value = vol.size * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-iterations/s (x particles)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "reference_step": "one oracle IFCM step of one particle over the full volume"},
        "cpu_baseline": {"value": value, "unit": "voxel-iterations/s (x particles)",
                         "cores": oracle.num_threads(), "kind": "oracle",
                         "host": host_info(oracle.num_threads()),
                         "sample": f"{args.steps} oracle IFCM steps of one particle each over the full volume"},
        "e2e": {"value": value, "unit": "voxel-iterations/s (x particles)",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    from paper_2002_01981_b200 import build as pbuild

    if rank == 0 or not os.path.exists(pbuild.LIB):
        pbuild.build()
    # one GPU per rank; PIFCM_BENCH_BACKEND=gloo (with ranks sharing a GPU)
    # only exercises the multi-rank code path, its numbers are not bench values
    backend = os.environ.get("PIFCM_BENCH_BACKEND", "nccl")
    dev_index = local_rank if backend == "nccl" else local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device(f"cuda:{dev_index}")
    dist = None
    if world > 1:
        import torch.distributed as tdist
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group(backend)
        dist = tdist
    ctx = Context(dev_index)
    c5 = args.workload == "C5"
    c2 = args.workload == "C2"
    c4 = args.workload == "C4"
    vol = _volume(args.workload)
    nz, ny, nx = vol.shape
    # C5: P = 64 as configured.  The CHAINED slot pool is 2P + 1 slab states
    # (129 x 2.16 GB at one GPU); where that does not fit, the particles are
    # evaluated in batches of eval_batch states over P + eval_batch + 1 slots
    # (bit-identical results, pifcm_pso_cfg.eval_batch)
    Pw = 64 if c5 else (20 if c2 else P)
    Pw = _env_int("PIFCM_BENCH_P", Pw)  # test hook (a smaller swarm), reported in config
    eval_batch = 0
    if c5:
        slot = (-(-nz // world) + 2) * ny * nx * 16
        free, _ = torch.cuda.mem_get_info(dev)
        avail = free - 8 * slot - (2 << 30)  # slab IFCM states, x, volume, labels, records
        if (2 * Pw + 1) * slot > avail:
            eval_batch = max(1, int(avail // slot) - Pw - 1)
    workload = WORKLOAD_C5.format(P=Pw) if c5 else (WORKLOAD_C2 if c2 else (WORKLOAD_C4 if c4 else WORKLOAD))
    cfg = IfcmConfig(C=C, m=2.0, q_mode=0, eps=1e-5, max_iter=100)
    pso = PsoConfig(P=Pw, ring_k=1, max_gen=GENS, patience=0, seed=12345, eval_batch=eval_batch)
    vol_d = torch.as_tensor(vol, device=dev)
    vol_h = torch.as_tensor(vol).pin_memory()
    lab_h = torch.empty(vol.shape, dtype=torch.uint8).pin_memory()
    stream = torch.cuda.current_stream(dev)

    if c5:
        from paper_2002_01981_b200.dist import SlabSegmenter
        seg = SlabSegmenter(ctx, cfg, pso, (nz, ny, nx), dist)

        def step():
            return seg.segment(vol_d)

        def step_host():
            rep = seg.segment(vol_h)
            lab_h.copy_(seg.labels, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return rep
    elif world > 1:
        from paper_2002_01981_b200.dist import ShardedSegmenter
        seg = ShardedSegmenter(ctx, cfg, pso, (nz, ny, nx), dist)

        def step():
            return seg.segment(vol_d)

        def step_host():
            return seg.segment_host(vol_h, lab_h)
    else:
        ws = ctx.workspace(nx, ny, nz, cfg, pso)
        lab_d = torch.empty(vol.shape, dtype=torch.uint8, device=dev)

        def step():
            return ctx.segment(vol_d, cfg, pso, ws=ws)[2]

        def step_host():
            return ctx.segment_host(vol_h, cfg, pso, ws, lab_h)

    if c4:  # one step = the whole batch of 16 volumes, one segmentation each
        from inputs import config_volume
        vols = [config_volume("C4", k=k)[0] for k in range(16)]
        vols_d = [torch.as_tensor(v, device=dev) for v in vols]
        vols_h = [torch.as_tensor(v).pin_memory() for v in vols]
        one_dev, one_host = step, step_host

        def _merge(rs):
            out = dict(rs[-1])
            out["units"] = sum(Pw * r["generations"] + r["final_iters"] for r in rs)
            out["t_pso"] = sum(r["t_pso"] for r in rs)
            out["t_total"] = sum(r["t_total"] for r in rs)
            return out

        def step():
            nonlocal vol_d
            rs = []
            for v in vols_d:
                vol_d = v
                rs.append(one_dev())
            return _merge(rs)

        def step_host():
            nonlocal vol_h
            rs = []
            for v in vols_h:
                vol_h = v
                rs.append(one_host())
            return _merge(rs)

    # voxel-iterations done per voxel: the PSO's P x generations and the final
    # IFCM's iterations.  The FCM start of a u8 volume runs on its <= 256-value
    # histogram (R24), not on the voxels, so its iterations are not counted
    # (reported separately as config.fcm_iters).
    def units(r):
        return r["units"] if "units" in r else Pw * r["generations"] + r["final_iters"]

    # ---- warm-up (the clock sampler starts here so it samples by the timed region)
    clocks = ClockSampler(dev_index) if rank == 0 else None
    if clocks:
        clocks.start()
    rep = None
    for _ in range(args.warmup):
        rep = step()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device-resident input
    ctx.timing_enable(True)
    l0 = ctx.launch_count()
    barrier()
    if clocks:
        clocks.mark()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    vp_total = 0.0
    reps = []
    for _ in range(args.steps):
        rep = step()
        reps.append(rep)
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop() if clocks else None
    launches = ctx.launch_count() - l0
    k_ms, k_n, k_bytes = ctx.timing_read(batched=True)     # PSO generations: P states per launch
    s_ms, s_n, s_bytes = ctx.timing_read(batched=False)    # final IFCM: one state per launch
    ctx.timing_enable(False)
    for r in reps:
        vp = nx * ny * nz * units(r)
        vp_total += vp
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = vp_total / (ms_max * 1e-3)

    # ---- e2e: host buffers through the public C-ABI call (H2D + D2H inside)
    barrier()
    h0 = torch.cuda.Event(enable_timing=True)
    h1 = torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    vp_e2e = 0.0
    for _ in range(args.steps):
        r = step_host()
        vp_e2e += nx * ny * nz * units(r)
    h1.record(stream)
    barrier()
    te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = vp_e2e / (float(te.item()) * 1e-3)

    dump = os.environ.get("PIFCM_BENCH_DUMP")  # test hook: the last e2e step's labels and (lambda*, xi*)
    if dump and rank == 0:
        np.savez(dump, labels=lab_h.numpy(), lam_xi=np.array([r["lambda"], r["xi"]]),
                 final_iters=np.array(r["final_iters"]))
    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    hbm, hbm_kind = _peaks()
    achieved = (k_bytes / k_n) / ((k_ms / k_n) * 1e-3) / 1e9 if k_n else None
    traffic = None
    ncu_instr = None
    if not c5 and not c2:  # the committed ncu capture is of the C3 P = 32 launch
        try:
            with open(PROFILE_SUMMARY) as f:
                summ = json.load(f)
            traffic = summ.get("dram_bytes_per_launch")
            ncu_instr = summ.get("instructions_per_vp")
        except Exception:
            pass
    # The kernel's binding resource is the FP32 pipe, not HBM:
    # the same launches against the FP32 lane-instruction peak, with SURVEY
    # §8(d)'s algorithmic count of 245 + 52/P FP32 instructions per vp
    # (an FMA counts once; H 78, F 112, g / G 52 shared by the P particles of
    # a launch, Eq. 4 / 2 / 3 / 1 ~53) and the peak 148 SMs x 128 lanes x the
    # max SM clock (B200_PROFILING: 1965 MHz).
    alu_view = None
    if k_n:
        if c5:  # every slab launch holds all particles on this rank's voxels
            p_launch = float(Pw)
            vox = (k_bytes / k_n) / (32.0 * Pw + 4.0)
        else:   # whole volume, this rank's particles
            vox = float(nx * ny * nz)
            p_launch = (k_bytes / k_n - 4.0 * vox) / (32.0 * vox)
        # (2D, 8 neighbours: SURVEY 8(d) counts ~110)
        instr_per_vp = 245.0 + 52.0 / max(p_launch, 1.0) if nz > 1 else 110.0
        vp_per_s = p_launch * vox / ((k_ms / k_n) * 1e-3)
        peak_alu = 148 * 128 * 1.965e9 / 1e12
        alu_view = {"bound": "alu", "achieved": vp_per_s * instr_per_vp / 1e12, "peak": peak_alu,
                    "unit": "T FP32 lane-instructions/s", "frac": vp_per_s * instr_per_vp / 1e12 / peak_alu,
                    "alg_instr_per_vp": instr_per_vp, "peak_kind": "derived (148 SM x 128 FP32 lanes x 1965 MHz)"}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline_measure(vol, budget_s=args.cpu_budget, P=Pw)
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "error": str(e), "kind": "oracle"}
    last = reps[-1]
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "voxel-iterations/s (x particles)",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {
            "workload": workload,
            "volume": [nx, ny, nz], "C": C, "P": Pw, "generations": GENS, "m": 2.0,
            "q_mode": "literal", "eps": 1e-5, "fitness": "chained",
            "parallelism": f"z-slabs/{world}" if c5 else f"particles/{world}",
            "l2": ("inputs larger than L2 (the membership slot pool is "
                   f"{((Pw + eval_batch + 1) if eval_batch else (2 * Pw + 1)) * nx * ny * nz * 16 / world / 1e9:.1f}"
                   f" GB per GPU; every generation streams {Pw * nx * ny * nz * 32 / 1e9:.1f} GB)"),
            "eval_batch": eval_batch,
            "pso_wall_ms": last["t_pso"] * 1e3, "segment_wall_ms": last["t_total"] * 1e3,
            # the segmentation's phases (CUDA events inside the library)
            "phases_ms": {k: last[k] * 1e3 for k in ("t_norm", "t_init", "t_pso", "t_final") if k in last},
            "fcm_iters": last["fcm_iters"], "final_iters": last["final_iters"],
            "lambda_star": last["lambda"], "xi_star": last["xi"],
        },
        **({"paper_context": {"what": "PAPER:250 Table 7: 3DPIFCM-GPU on a TITAN X, whole algorithm, 854x854 "
                                      "(particles / generations not stated)", "seconds": PAPER_C2_SECONDS,
                              "ours_seconds": ms_max / args.steps * 1e-3}} if c2 else {}),
        "roofline": {
            "bound": "hbm",
            "kernel": ("k_step_stencil, one launch = one PSO generation (all P particles' fused IFCM steps"
                       + (", this rank's slab)" if c5 else ")")),
            "achieved": achieved,
            "peak": hbm,
            "peak_kind": hbm_kind,
            "unit": "GB/s",
            "frac": (achieved / hbm) if achieved else None,
            "traffic": traffic,
            "alg_bytes_per_launch": (k_bytes / k_n) if k_n else None,
            "alg_bytes_per_unit": "32 B per voxel x particle (fp32 AoS-C4 membership row read + write) + 4 B per voxel of intensities",
            "avg_launch_ms": (k_ms / k_n) if k_n else None,
            "launches": k_n,
            "share_of_step": (k_ms / ms) if ms else None,
            "alu": alu_view,
            # smsp__inst_executed / (N_vox P) of the same launch, from the committed ncu capture
            "ncu_instr_per_vp": ncu_instr,
            "single_state_launches": {
                "what": "final IFCM (P = 1) launches of the same kernel",
                "launches": s_n, "avg_launch_ms": (s_ms / s_n) if s_n else None,
                "achieved_GBs": ((s_bytes / s_n) / ((s_ms / s_n) * 1e-3) / 1e9) if s_n else None,
                "share_of_step": (s_ms / ms) if ms else None,
            },
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "voxel-iterations/s (x particles)",
                "h2d_bytes_per_step": int(vol.size) * (16 if c4 else 1),
                "d2h_bytes_per_step": int(vol.size) * (16 if c4 else 1)},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--workload", default="C3", choices=["C3", "C2", "C4", "C5"],
                    help="C3 (default, the BASELINE metric's config), C2 (854x854 2D, the paper's Table 7 "
                         "image), C4 (16 C3-shaped volumes per step) or C5 (512^3, z-slab sharded)")
    args = ap.parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
