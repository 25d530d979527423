"""profiles/kstep_summary.json from an `ncu --set full` report of one P = 32
k_step_stencil launch (tools/round_profile.sh).  Runs here, no GPU.

    python tools/kstep_summary.py gpurun_out/kstep_r01b.ncu-rep > profiles/kstep_summary.json
"""
import collections
import csv
import json
import re
import subprocess
import sys

rep = sys.argv[1]
NVOX = 181 * 217 * 181
P = 32
ALG = 32.0 * NVOX * P + 4.0 * NVOX  # bench.py's algorithmic bytes per launch


def raw():
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]

    def g(name):
        x = v[h.index(name)].replace(",", "")
        return float(x)
    return h, v, g


h, v, g = raw()
unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
units = rows[1]


def bytes_of(name):
    return g(name) * unit.get(units[h.index(name)], 1.0)


rd, wr = bytes_of("dram__bytes_read.sum"), bytes_of("dram__bytes_write.sum")
dur_u = units[h.index("gpu__time_duration.sum")]
dur_ms = g("gpu__time_duration.sum") * {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6,
                                        "nsecond": 1e-6}.get(dur_u, 1.0)
stalls = {}
for k in h:
    m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
    if m and v[h.index(k)] not in ("", "n/a"):
        val = float(v[h.index(k)])
        if val > 0.05:
            stalls[m.group(1)] = round(val, 3)

# SASS opcode mix from the source page (executed warp instructions per opcode)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
sh = srows[1]
si, ei = sh.index("Source"), sh.index("Instructions Executed")
mix = collections.Counter()
for r in srows[2:]:
    if len(r) <= ei:
        continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si].strip())
    if m and r[ei]:
        mix[m.group(2)] += int(r[ei])
tot = sum(mix.values())
per_vp = {op: round(n * 32 / (NVOX * P), 1) for op, n in mix.most_common(12)}

out = {
    "source": f"{rep}: ncu --set full --clock-control none --import-source on, k_step_stencil<C=4,m=2>, one "
              "launch = one PSO generation (P=32 particles) of the C3 workload (tools/profile_step.py eval 2, "
              "second launch)",
    "kernel": v[h.index("Kernel Name")],
    "duration_ms_under_ncu": dur_ms,
    "dram_read_GB": rd / 1e9,
    "dram_write_GB": wr / 1e9,
    "dram_bytes_per_launch": rd + wr,
    "alg_bytes_per_launch": ALG,
    "traffic_over_alg": (rd + wr) / ALG,
    "dram_throughput_pct_of_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "sm_throughput_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "fma_pipe_active_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_active_pct": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": g("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": g("launch__registers_per_thread"),
    "warp_instructions": float(tot),
    "instructions_per_vp": tot * 32 / (NVOX * P),
    "sass_per_vp_top12": per_vp,
    "stalls_per_issue": stalls,
}
print(json.dumps(out, indent=1))
