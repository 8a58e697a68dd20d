"""Attribute executed instructions / stall samples to CUDA source lines from
`ncu -i rep --page source --csv --print-source cuda,sass` (development tool).

    python tools/sass_lines.py mix.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
ins, smp, txt, fil = defaultdict(float), defaultdict(float), {}, None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fil = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    line = r[0]
    if not line:  # SASS rows under a source line: the line row already sums them
        continue
    txt[(fil, line)] = r[1]
    try:
        n = float(r[7] or 0)
        s = float(r[4] or 0)
    except ValueError:
        continue
    ins[(fil, line)] += n
    smp[(fil, line)] += s
tn, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for k in sorted(ins, key=lambda k: -(ins[k] / tn + smp[k] / ts))[:top]:
    print(f"{100 * ins[k] / tn:5.1f}% inst {100 * smp[k] / ts:5.1f}% stall {k[0]}:{k[1]:>4s} "
          f"{txt.get(k, '').strip()[:90]}")
