"""u8 / f32 strip pipeline rebuilt in torch streams (development tool): H2D
strips on s_in, the fused kernel per strip on s_k, D2H strips on s_out, with
and without the kernels, to see what serializes the copy engines."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, synth  # noqa: E402

H, W = 2160, 3840
dev = torch.device("cuda", 0)
c = synth.make_case(0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
tables = device.pack_tables(device.reconstruct(T(c.u)[None], T(c.s)[None], T(c.vt)[None]), T(c.lw)[None],
                            T(c.lb)[None], T(c.grid_planes)[None], T(c.gw)[None], T(c.gb)[None])
h_in = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
h_in.copy_(torch.from_numpy((c.rgb.transpose(1, 2, 0) * 255).astype(np.uint8)))
h_out = torch.empty_like(h_in).pin_memory()
d_in = torch.empty((1, H, W, 3), dtype=torch.uint8, device=dev)
d_out = torch.empty_like(d_in)
s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(bounds, kernel, mode="3s"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        e0.record(s_in)
        s_out.wait_event(e0)
        s_k.wait_event(e0)
        for r0, r1 in zip(bounds, bounds[1:]):
            with torch.cuda.stream(s_in):
                d_in[0, r0:r1].copy_(h_in[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
            s_k.wait_event(ev)
            with torch.cuda.stream(s_k):
                if kernel:
                    device.apply_io(d_in[:, r0:r1], tables, in_fmt="u8", out_fmt="u8", out=d_out[:, r0:r1],
                                    y0=r0, h_total=H)
            ev2 = torch.cuda.Event()
            ev2.record(s_k)
            s_out.wait_event(ev2)
            with torch.cuda.stream(s_out):
                h_out[r0:r1].copy_(d_out[0, r0:r1], non_blocking=True)
        s_in.wait_stream(s_out)
        e1.record(s_in)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[4]


for n in (2, 4, 6):
    unit = H // n
    b = [0] + [min(H, unit // 4 + i * unit) for i in range(n)] + [H]
    b = sorted(set(b))
    print(f"strips {len(b) - 1}: copies only {run(b, False):.3f} ms   with kernels {run(b, True):.3f} ms",
          file=sys.stderr)

# the library's own host pipeline on the same pinned buffers
import time  # noqa: E402

from paper_2508_16121_b200 import transform  # noqa: E402
from paper_2508_16121_b200.core_types import GridSet, GridWeights, Lut2DSet, LutWeights  # noqa: E402

planes = device.reconstruct(T(c.u)[None], T(c.s)[None], T(c.vt)[None])[0].cpu().numpy()
args = (h_in.numpy(), Lut2DSet(planes), LutWeights(c.lw, c.lb), GridSet(c.grid_planes), GridWeights(c.gw, c.gb))
for _ in range(3):
    transform.enhance_payload(*args, out=h_out.numpy())
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    transform.enhance_payload(*args, out=h_out.numpy())
    ts.append(time.perf_counter() - t0)
print(f"enhance_payload (C++ pipeline, same buffers): {1e3 * np.median(ts):.3f} ms", file=sys.stderr)
