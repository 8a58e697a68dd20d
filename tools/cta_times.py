"""Per-CTA start/end times of the fused forward (development tool; needs a
build with -DFWD_DBG_TIMES, e.g. tools/build_variant.py times -DFWD_DBG_TIMES)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_16121_b200 import device, synth  # noqa: E402

dev = torch.device("cuda", 0)
c = synth.make_case(0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
planes = device.reconstruct(T(c.u), T(c.s), T(c.vt))
tables = device.pack_tables(planes, T(c.lw), T(c.lb), T(c.grid_planes), T(c.gw), T(c.gb))
x = T(c.rgb)[None]
flag = torch.zeros(2 + 4 * 148, dtype=torch.int32, device=dev)
for _ in range(5):
    device.apply(x, tables, nonfinite=flag)
torch.cuda.synchronize()
t = flag[2:].cpu().numpy().view(np.uint64).reshape(148, 2).astype(np.float64)
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
order = np.argsort(end)
print(f"start: min {start.min():.2f} max {start.max():.2f} us")
print(f"end:   min {end.min():.2f} median {np.median(end):.2f} max {end.max():.2f} us")
print("busy (end-start) per CTA: min %.2f max %.2f" % ((end - start).min(), (end - start).max()))
rows = [(2160 * (i + 1)) // 148 - (2160 * i) // 148 for i in range(148)]
for r in (14, 15):
    sel = [i for i in range(148) if rows[i] == r]
    print(f"CTAs with {r} rows: n={len(sel)} end median {np.median(end[sel]):.2f} max {end[sel].max():.2f}")
