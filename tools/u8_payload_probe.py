"""u8 host path from successive input payload buffers (development tool):
fill method (multi-threaded torch copy_ / single-thread numpy assignment) and
buffer lifetime (kept / dropped before the next).  Measured: torch-filled
inputs 1.3-1.7 ms per 4K frame, numpy-filled 0.82 ms (the DMA reads snoop the
lines the copy threads left dirty in their private caches); huge-page backed
buffers (mmap + MADV_HUGEPAGE + cudaHostRegister) made no difference."""
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
factors = SvdLut(c.u, c.s, c.vt)
lw, grids, gw = LutWeights(c.lw, c.lb), GridSet(c.grid_planes), GridWeights(c.gw, c.gb)
pay = np.floor(np.clip(c.rgb.transpose(1, 2, 0), 0, 1) * 255 + 0.5).astype(np.uint8)
q = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True).numpy()
keep = []


def timed(pin8):
    for _ in range(3):
        transform.enhance_payload(pin8, svd.reconstruct_lut(factors), lw, grids, gw, out=q)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        transform.enhance_payload(pin8, svd.reconstruct_lut(factors), lw, grids, gw, out=q)
        ts.append(time.perf_counter() - t0)
    return 1e3 * np.median(ts)


for alloc in ("torch",):
    for fill in ("torch", "numpy"):
        for life in ("drop", "keep"):
            res = []
            for _ in range(3):
                t = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
                a = t.numpy()
                if fill == "torch":
                    t.copy_(torch.from_numpy(pay))
                else:
                    a[...] = pay
                res.append(timed(a))
                if life == "keep":
                    keep.append((t, a))
                del t, a
            print(f"{alloc:8s} fill {fill:6s} {life}: " + " ".join(f"{v:.3f}" for v in res) + " ms",
                  file=sys.stderr)
