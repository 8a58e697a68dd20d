"""Sample-format variants of the fused apply at 4K (development tool):
device kernel time for f32 / u8 / u16be in+out, and the host entry
transform.enhance_payload (PNM payload in, payload out, PCIe included)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, synth, transform  # noqa: E402
from paper_2508_16121_b200.core_types import GridSet, GridWeights, Lut2DSet, LutWeights  # noqa: E402

H, W = 2160, 3840
dev = torch.device("cuda", 0)
c = synth.make_case(0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
planes = device.reconstruct(T(c.u), T(c.s), T(c.vt))
tables = device.pack_tables(planes, T(c.lw), T(c.lb), T(c.grid_planes), T(c.gw), T(c.gb))
img16 = np.ascontiguousarray(np.round(c.rgb.transpose(1, 2, 0) * 65535).astype(np.uint16))
img8 = np.ascontiguousarray((img16 >> 8).astype(np.uint8))
be = np.ascontiguousarray(img16.astype(">u2")).view(np.uint8).reshape(H, W, 6)
inputs = {"f32": T(c.rgb)[None], "u8": T(img8)[None], "u16be": T(be)[None]}
for fmt, x in inputs.items():
    xs = [x] + [torch.roll(x, 64 * i, dims=2).contiguous() for i in range(1, 4)]
    outs = [device.apply_io(xi, tables, fmt, fmt) for xi in xs]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(40):
        device.apply_io(xs[i % 4], tables, fmt, fmt, out=outs[i % 4])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 40
    bpp = {"f32": 24, "u8": 6, "u16be": 12}[fmt]
    print(f"kernel {fmt:6s} in/out  {us:7.2f} us  {H * W / us:9.0f} MP/s  {bpp * H * W / us / 1e3:7.1f} GB/s ({bpp} B/px)")

lut, lw = Lut2DSet(planes[0].cpu().numpy()), LutWeights(c.lw, c.lb)
grids, gw = GridSet(c.grid_planes), GridWeights(c.gw, c.gb)
pin8 = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
pin8.copy_(torch.from_numpy(img8))
pin16 = torch.empty(H * W * 6, dtype=torch.uint8, pin_memory=True).numpy().view(">u2").reshape(H, W, 3)
pin16[...] = img16
for name, payload in (("u8", pin8.numpy()), ("u16", pin16)):
    transform.enhance_payload(payload, lut, lw, grids, gw)
    t0 = time.perf_counter()
    for _ in range(10):
        transform.enhance_payload(payload, lut, lw, grids, gw)
    ms = (time.perf_counter() - t0) * 100
    print(f"host enhance_payload {name:4s}  {ms:7.3f} ms  {H * W / ms / 1e3:9.0f} MP/s")
