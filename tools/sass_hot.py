"""Per-instruction execution counts of an ncu source page (--print-source sass
--csv): instruction mix per voxel-particle by region, the hottest stall sites.
    python tools/sass_hot.py gpurun_out/sass_X.csv [vp]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
vp = float(sys.argv[2]) if len(sys.argv) > 2 else 181 * 217 * 181 * 32
iA, iS, iE, iSamp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    n = float(r[iE] or 0)
    src = r[iS].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    ins.append((int(r[iA], 16), op, n, float(r[iSamp] or 0), src))
base = ins[0][0]
tot = sum(n for _, _, n, _, _ in ins)
print(f"warp instructions {tot:.4g}, thread-instr/vp {tot * 32 / vp:.1f}")
mix = collections.Counter()
for _, op, n, _, _ in ins:
    mix[op.split(".")[0]] += n * 32 / vp
print("mix/vp:", ", ".join(f"{k} {v:.1f}" for k, v in mix.most_common(30)))
# regions: contiguous blocks of instructions with equal execution count
blocks = []
for a, op, n, s, src in ins:
    if blocks and blocks[-1][2] == n:
        blocks[-1][1] = a
        blocks[-1][3] += 1
        blocks[-1][4] += s
        blocks[-1][5][op.split(".")[0]] += 1
    else:
        blocks.append([a, a, n, 1, s, collections.Counter({op.split(".")[0]: 1})])
print("blocks by instr/vp:")
for b in sorted(blocks, key=lambda b: -b[2] * b[3])[:25]:
    print(f"  {b[0]-base:#07x}-{b[1]-base:#07x} n={b[2]:.4g} len={b[3]} instr/vp={b[2]*b[3]*32/vp:.2f} samples={b[4]:.0f} "
          + " ".join(f"{k}:{v}" for k, v in b[5].most_common(8)))
