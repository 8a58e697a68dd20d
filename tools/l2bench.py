"""Forward vs fused-L2 forward on the config-5 batch (8 x 1080p) (development tool)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, synth  # noqa: E402

dev = torch.device("cuda", 0)
B, H, W = 8, 1080, 1920
case = synth.make_batch(list(range(B)), h=H, w=W)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
tables = device.pack_tables(device.reconstruct(T(case.u), T(case.s), T(case.vt)), T(case.lw), T(case.lb),
                            T(case.grid_planes), T(case.gw), T(case.gb))
x = T(case.rgb)
tgt = x.clamp_min(0) ** 0.8
out = torch.empty_like(x)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


px = B * H * W
for name, fn in (("forward f32", lambda: device.apply(x, tables, out=out)),
                 ("forward + L2 epilogue", lambda: device.apply_l2(x, tgt, tables))):
    us = timed(fn)
    print(f"{name:24s} {us:8.1f} us  {px / us:9.0f} MP/s", file=sys.stderr)
