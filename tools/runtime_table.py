"""Multi-stage vs fused runtime on B200 (the paper's tab:runtime comparison,
SURVEY.md §8(f) row 3), device-resident inputs, CUDA-event timing of 20
calls replayed from one CUDA graph:

  fused fast      svdlut fused fp32 kernel (product path)
  fused exact     f64 op-for-op kernel (bitwise equal to the reference)
  multi-stage     slice_grid2d + apply_lut2d + combine_slices (f64 stage kernels,
                  every intermediate raster materialized in HBM)
  3D LUT          trilinear 3D-LUT baseline, d = 33 (f64, reference order)

    python tools/runtime_table.py [--out profiles/runtime_table_r01.txt]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import device, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)[None]  # noqa: E731
lines = [f"{'resolution':>11s} {'fused fast':>12s} {'fused exact':>12s} {'multi-stage':>12s} "
         f"{'3D LUT d=33':>12s}   (us per frame; MP/s of the fused fast path)"]
for h, w in ((480, 720), (1080, 1920), (2160, 3840)):
    c = synth.make_case(0, h=h, w=w)
    x = T(c.rgb)
    planes = device.reconstruct(T(c.u), T(c.s), T(c.vt))
    lw, lb, gp, gw, gb = T(c.lw), T(c.lb), T(c.grid_planes), T(c.gw), T(c.gb)
    tables = device.pack_tables(planes, lw, lb, gp, gw, gb)
    cubes = T(np.random.default_rng(1).random((3, 33, 33, 33), dtype=np.float32))
    runs = {
        "fast": lambda: device.apply(x, tables),
        "exact": lambda: device.apply_exact(x, planes, lw, lb, gp, gw, gb),
        "multi": lambda: device.combine_slices(device.apply_lut2d(x, planes, lw, lb),
                                               device.slice_grids(x, gp, gw, gb)),
        "lut3d": lambda: device.apply_lut3d(x, cubes),
    }
    res = {}
    for name, fn in runs.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        # 20 calls captured in one CUDA graph: device time per frame, without
        # the ~20 us of Python per call that dominates small frames
        reps = 20
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            for _ in range(reps):
                fn()
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) * 1e3 / reps
    lines.append(f"{h:>5d}x{w:<5d} {res['fast']:12.1f} {res['exact']:12.1f} {res['multi']:12.1f} "
                 f"{res['lut3d']:12.1f}   ({h * w / res['fast']:.0f} MP/s)")
text = "\n".join(lines)
print(text)
if a.out:
    open(a.out, "w").write(text + "\n")
