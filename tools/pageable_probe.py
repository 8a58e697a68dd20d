"""fused_enhance from a pageable numpy image vs a page-locked one (development tool)."""
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

H, W = 2160, 3840
c = synth.make_case(0)
luts = svd.reconstruct_lut(SvdLut(c.u, c.s, c.vt))
args = (luts, LutWeights(c.lw, c.lb), GridSet(c.grid_planes), GridWeights(c.gw, c.gb))
pageable = np.array(c.rgb, copy=True)
pin = torch.empty((3, H, W), dtype=torch.float32, pin_memory=True).numpy()
pin[...] = c.rgb
for name, arr in (("pinned", pin), ("pageable", pageable)):
    img = Image(W, H, arr)
    for _ in range(3):
        transform.fused_enhance(img, *args)
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        transform.fused_enhance(img, *args)
        ts.append(time.perf_counter() - t0)
    print(f"{name:9s} input: {1e3 * np.median(ts):.3f} ms", file=sys.stderr)
