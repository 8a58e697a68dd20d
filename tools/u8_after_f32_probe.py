"""Does the u8 payload path slow down after the f32 host path ran in the same
process (development tool)?"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, svd, synth, transform  # noqa: E402
from paper_2508_16121_b200.core_types import (GridSet, GridWeights, Image, Lut2DSet, LutWeights,  # noqa: E402
                                              SvdLut)

H, W = 2160, 3840
c = synth.make_case(0)
factors = SvdLut(c.u, c.s, c.vt)
lw, grids, gw = LutWeights(c.lw, c.lb), GridSet(c.grid_planes), GridWeights(c.gw, c.gb)
pin8 = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
pin8.copy_(torch.from_numpy((c.rgb.transpose(1, 2, 0) * 255).astype(np.uint8)))
q = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True).numpy()


def u8(tag):
    for _ in range(3):
        transform.enhance_payload(pin8.numpy(), svd.reconstruct_lut(factors), lw, grids, gw, out=q)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        transform.enhance_payload(pin8.numpy(), svd.reconstruct_lut(factors), lw, grids, gw, out=q)
        ts.append(time.perf_counter() - t0)
    print(f"{tag}: u8 {1e3 * np.median(ts):.3f} ms", file=sys.stderr)


u8("fresh process")
pin = torch.empty((3, H, W), dtype=torch.float32, pin_memory=True)
pin.copy_(torch.from_numpy(c.rgb))
img = Image(W, H, pin.numpy())
for _ in range(14):
    y = transform.fused_enhance(img, svd.reconstruct_lut(factors), lw, grids, gw)
u8("after 14 f32 calls")
del y
torch.cuda.synchronize()
big = [torch.empty(128 << 20, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
u8("with 512 MB more pinned")
x = torch.empty(760 << 20, dtype=torch.uint8, device="cuda")
u8("with 760 MB device tensor")
import pynvml  # noqa: E402

pynvml.nvmlInit()
u8("after nvmlInit")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
tables = device.pack_tables(device.reconstruct(T(c.u)[None], T(c.s)[None], T(c.vt)[None]), T(c.lw)[None],
                            T(c.lb)[None], T(c.grid_planes)[None], T(c.gw)[None], T(c.gb)[None])
xin = T(c.rgb)[None]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    device.apply(xin, tables)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        yo = device.apply(xin, tables)
for _ in range(20):
    g.replay()
torch.cuda.synchronize()
u8("after graph replays")
