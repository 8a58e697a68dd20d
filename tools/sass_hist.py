"""Per-opcode histogram of executed warp instructions / stall samples from
`ncu -i rep --page source --csv --print-source sass` output (development tool).

    python tools/sass_hist.py sass.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ins, smp, thr = defaultdict(float), defaultdict(float), defaultdict(float)
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    n = float(r[ix["Instructions Executed"]] or 0)
    ins[op] += n
    thr[op] += float(r[ix["Thread Instructions Executed"]] or 0)
    smp[op] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(ins.values()) or 1
stot = sum(smp.values()) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"{'opcode':28s} {'warp-inst':>12s} {'%':>6s} {'thr/inst':>8s} {'stall%':>7s}")
for op, n in sorted(ins.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{op:28s} {n:12.0f} {100 * n / tot:6.2f} {thr[op] / max(n, 1):8.1f} {100 * smp[op] / stot:7.2f}")
print(f"total {tot:.0f}")
