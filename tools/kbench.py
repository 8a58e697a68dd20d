"""Kernel-level timing of the fused forward (development tool).

    [SVDLUT_LIB=<variant .so>] python tools/kbench.py [--reps 50] [--only smooth|uniform] [--once]

Prints one line per workload: kernel µs (CUDA events over `reps` launches
rotating 4 buffer sets), GB/s at 24 B/pixel, fraction of the measured HBM copy
peak.  --once launches the kernel once (for ncu captures).
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--only", default=None)
ap.add_argument("--once", action="store_true")
ap.add_argument("--h", type=int, default=2160)
ap.add_argument("--w", type=int, default=3840)
a = ap.parse_args()

dev = torch.device("cuda", 0)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
H, W = a.h, a.w
work = {"smooth": lambda: synth.make_case(0, h=H, w=W),
        "uniform": lambda: synth.uniform_case(0, H, W)}
for name, mk in work.items():
    if a.only and name != a.only:
        continue
    case = mk()
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    planes = device.reconstruct(T(case.u), T(case.s), T(case.vt))
    tables = device.pack_tables(planes, T(case.lw), T(case.lb), T(case.grid_planes), T(case.gw),
                                T(case.gb))
    base = T(case.rgb)[None]
    ins = [base] + [torch.roll(base, 17 * i, 3).contiguous() for i in range(1, 4)]
    outs = [torch.empty_like(base) for _ in range(4)]
    if a.once:
        device.apply(ins[0], tables, out=outs[0])
        torch.cuda.synchronize()
        print(f"{name} launched once")
        continue
    for i in range(5):
        device.apply(ins[i % 4], tables, out=outs[i % 4])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(a.reps):
        device.apply(ins[i % 4], tables, out=outs[i % 4])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    gbs = 24 * H * W / (us * 1e-6) / 1e9
    print(f"{os.environ.get('SVDLUT_LIB', 'default')} {name:8s} {H}x{W} {us:8.2f} us  {gbs:7.1f} GB/s  "
          f"frac={gbs / peak:.3f}  {H * W / us:.0f} MP/s")
