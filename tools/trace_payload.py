"""One traced transform.enhance_payload call (SVDLUT_TRACE=1 prints the strip
timeline) for a 4K u8 payload (development tool)."""
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

c = synth.make_case(0)
planes = device.reconstruct(*(torch.from_numpy(a).cuda() for a in (c.u, c.s, c.vt)))[0].cpu().numpy()
pin = torch.empty((2160, 3840, 3), dtype=torch.uint8, pin_memory=True)
pin.copy_(torch.from_numpy(np.ascontiguousarray((c.rgb.transpose(1, 2, 0) * 255).astype(np.uint8))))
args = (pin.numpy(), Lut2DSet(planes), LutWeights(c.lw, c.lb), GridSet(c.grid_planes),
        GridWeights(c.gw, c.gb))
for _ in range(3):
    transform.enhance_payload(*args)
t0 = time.perf_counter()
transform.enhance_payload(*args)
print(f"one call {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr)
