"""One traced transform.fused_enhance call on a 4K f32 frame in page-locked
memory (SVDLUT_TRACE=1 prints the strip timeline; development tool), plus
the bare concurrent H2D || D2H copy time of the same bytes."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import svd, synth, transform  # noqa: E402
from paper_2508_16121_b200.core_types import GridSet, GridWeights, Image, LutWeights, SvdLut  # noqa: E402

c = synth.make_case(0)
H, W = c.rgb.shape[1:]
pin = torch.empty((3, H, W), dtype=torch.float32, pin_memory=True)
pin.numpy()[...] = c.rgb
img = Image(W, H, pin.numpy())
f, lw, g, gw = SvdLut(c.u, c.s, c.vt), LutWeights(c.lw, c.lb), GridSet(c.grid_planes), GridWeights(c.gw, c.gb)
for _ in range(5):
    transform.fused_enhance(img, svd.reconstruct_lut(f), lw, g, gw)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    transform.fused_enhance(img, svd.reconstruct_lut(f), lw, g, gw)
    ts.append(1e3 * (time.perf_counter() - t0))
print("reconstruct_lut + fused_enhance ms: " + " ".join(f"{t:.2f}" for t in ts), file=sys.stderr)
luts = svd.reconstruct_lut(f)
for name, fn in (("reconstruct_lut", lambda: svd.reconstruct_lut(f)),
                 ("fused_enhance", lambda: transform.fused_enhance(img, luts, lw, g, gw))):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn()
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{name} alone ms: " + " ".join(f"{t:.3f}" for t in sorted(ts)[:5]), file=sys.stderr)
os.environ["SVDLUT_TRACE"] = "1"
# bare duplex copies of the same bytes
d_in = torch.empty((3, H, W), dtype=torch.float32, device="cuda")
d_out = torch.empty((3, H, W), dtype=torch.float32, device="cuda")
h_out = torch.empty((3, H, W), dtype=torch.float32, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d_in.copy_(pin, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d_in.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"H2D||D2H {1e3 * (t1 - t0):.3f} ms   H2D alone {1e3 * (t2 - t1):.3f}   D2H alone {1e3 * (t3 - t2):.3f}",
          file=sys.stderr)
