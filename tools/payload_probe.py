"""Where does the PNM-payload e2e step go? (development tool)"""
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
from paper_2508_16121_b200.core_types import GridSet, GridWeights, LutWeights, SvdLut  # noqa: E402

H, W = 2160, 3840
c = synth.make_case(0)
pin = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
pin.copy_(torch.from_numpy(np.ascontiguousarray((c.rgb.transpose(1, 2, 0) * 255).astype(np.uint8))))
payload = pin.numpy()
f, lw = SvdLut(c.u, c.s, c.vt), LutWeights(c.lw, c.lb)
grids, gw = GridSet(c.grid_planes), GridWeights(c.gw, c.gb)
luts = svd.reconstruct_lut(f)
out = transform._pinned_payload((H, W, 3), 1)


def t(fn, n=10):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e3


print(f"pinned alloc 25MB   {t(lambda: transform._pinned_payload((H, W, 3), 1)):7.3f} ms")
print(f"reconstruct_lut     {t(lambda: svd.reconstruct_lut(f)):7.3f} ms")
print(f"payload, out given  {t(lambda: transform.enhance_payload(payload, luts, lw, grids, gw, out=out)):7.3f} ms")
print(f"payload, alloc      {t(lambda: transform.enhance_payload(payload, luts, lw, grids, gw)):7.3f} ms")
keep = []
print(f"payload, alloc+keep {t(lambda: keep.append(transform.enhance_payload(payload, luts, lw, grids, gw)) or keep.pop(0) if len(keep) > 1 else None):7.3f} ms")
