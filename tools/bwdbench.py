"""Config-5 style timing of the backward (development tool).

Batch of B smooth 1080p images: forward (pack + apply), L2 loss against
X^0.8, gY = 2(Y-T)/N, then svdlut_fused_bwd + reconstruct backward.
Prints µs per backward and the 36 B/pixel bandwidth it implies.
"""

import argparse
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
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--uniform", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
H, W = 1080, 1920
if a.uniform:
    cases = [synth.uniform_case(s, H, W) for s in range(a.batch)]
    case = synth.Case(*(np.stack([getattr(c, f) for c in cases]) for f in synth.Case.__dataclass_fields__))
else:
    case = synth.make_batch(list(range(a.batch)), h=H, w=W)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
t = {k: T(getattr(case, k)) for k in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
planes = device.reconstruct(t["u"], t["s"], t["vt"])
y = device.fused_forward(t["rgb"], planes, t["lw"], t["lb"], t["grid_planes"], t["gw"], t["gb"])
target = t["rgb"].clamp_min(0) ** 0.8
gy = 2.0 * (y - target) / y.numel()


def bwd():
    g = device.fused_backward(t["rgb"], gy, planes, t["lw"], t["grid_planes"], t["gw"])
    device.reconstruct_backward(t["u"], t["s"], t["vt"], g["dlut_planes"])
    return g


for _ in range(2):
    bwd()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(a.reps):
    bwd()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / a.reps
px = a.batch * H * W
print(f"backward batch={a.batch} {'uniform' if a.uniform else 'smooth'}: {us:9.1f} us  "
      f"{36 * px / (us * 1e-6) / 1e9:7.1f} GB/s (36 B/px)  {px / us:8.0f} MP/s")
