"""One config-5-shaped backward launch, then one one-pass training step
(svdlut_fused_l2_step, the same kernel with the forward folded in), for ncu
captures: -k regex:fused_bwd_kernel -c 1 takes the backward, -s 1 -c 1 the
training step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, synth  # noqa: E402

dev = torch.device("cuda", 0)
case = synth.make_batch([0, 1], h=1080, w=1920)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
t = {k: T(getattr(case, k)) for k in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
planes = device.reconstruct(t["u"], t["s"], t["vt"])
y = device.fused_forward(t["rgb"], planes, t["lw"], t["lb"], t["grid_planes"], t["gw"], t["gb"])
gy = 2.0 * (y - t["rgb"].clamp_min(0) ** 0.8) / y.numel()
g = device.fused_backward(t["rgb"], gy, planes, t["lw"], t["grid_planes"], t["gw"])
tables = device.pack_tables(planes, t["lw"], t["lb"], t["grid_planes"], t["gw"], t["gb"])
loss, g2 = device.fused_l2_step(t["rgb"], t["rgb"].clamp_min(0) ** 0.8, tables, planes, t["lw"], t["grid_planes"],
                                t["gw"])
torch.cuda.synchronize()
print("ok", float(g["dlw"].abs().sum()), float(g2["dlw"].abs().sum()))
