"""Break down the end-to-end host path (development tool).

Times: pinned H2D / D2H of one 4K image (1-D and 2-D copies), the
reference-facing reconstruct_lut and fused_enhance calls, and the C entry
svdlut_enhance_host alone.
"""

import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import _lib, svd, synth, transform  # noqa: E402
from paper_2508_16121_b200.core_types import GridSet, GridWeights, Image, LutWeights, SvdLut  # noqa: E402

H, W = 2160, 3840
dev = torch.device("cuda", 0)
case = synth.make_case(0)
pin_in = torch.empty((3, H, W), dtype=torch.float32, pin_memory=True)
pin_in.copy_(torch.from_numpy(case.rgb))
pin_out = torch.empty_like(pin_in).pin_memory()
d = torch.empty((3, H, W), dtype=torch.float32, device=dev)


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


nb = case.rgb.nbytes
ms = timeit(lambda: d.copy_(pin_in, non_blocking=True))
print(f"H2D pinned 1-D  {ms:7.3f} ms  {nb / ms / 1e6:6.1f} GB/s")
ms = timeit(lambda: pin_out.copy_(d, non_blocking=True))
print(f"D2H pinned 1-D  {ms:7.3f} ms  {nb / ms / 1e6:6.1f} GB/s")
s2 = torch.cuda.Stream()


def both():
    d.copy_(pin_in, non_blocking=True)
    with torch.cuda.stream(s2):
        pin_out.copy_(d2, non_blocking=True)


d2 = torch.empty_like(d)
ms = timeit(both)
print(f"H2D||D2H        {ms:7.3f} ms  {2 * nb / ms / 1e6:6.1f} GB/s (both directions)")

img = Image(W, H, pin_in.numpy())
factors = SvdLut(case.u, case.s, case.vt)
lw = LutWeights(case.lw, case.lb)
grids, gw = GridSet(case.grid_planes), GridWeights(case.gw, case.gb)
luts = svd.reconstruct_lut(factors)
print(f"reconstruct_lut {timeit(lambda: svd.reconstruct_lut(factors)):7.3f} ms")
print(f"fused_enhance   {timeit(lambda: transform.fused_enhance(img, luts, lw, grids, gw)):7.3f} ms")
print(f"alloc_raster    {timeit(lambda: transform._alloc_raster((3, H, W))):7.3f} ms")

L = _lib.load()
ctx = transform._host_ctx(0)
out = pin_out.numpy()
flag = ctypes.c_int(0)
P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
planes = np.ascontiguousarray(luts.planes)


def host_call():
    _lib.call("svdlut_enhance_host", ctx, P(img.data), H, W, P(planes), P(lw.w), P(lw.b), 33,
              P(grids.planes), P(gw.w), P(gw.b), 6, 17, P(out), 0, ctypes.byref(flag))


print(f"enhance_host    {timeit(host_call):7.3f} ms")

if os.environ.get("SVDLUT_STRIP_KB"):
    print(f"strip_kb={os.environ['SVDLUT_STRIP_KB']} enhance_host {timeit(host_call, 20):7.3f} ms")

if os.environ.get("PROBE_PIPE"):
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    flat_in, flat_d, flat_out = pin_in.view(-1), d.view(-1), pin_out.view(-1)

    def pipe(n):
        evs = []
        step = flat_in.numel() // n
        for i in range(n):
            sl = slice(i * step, (i + 1) * step if i < n - 1 else flat_in.numel())
            with torch.cuda.stream(s_in):
                flat_d[sl].copy_(flat_in[sl], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
            with torch.cuda.stream(s_out):
                s_out.wait_event(e)
                flat_out[sl].copy_(flat_d[sl], non_blocking=True)
        torch.cuda.synchronize()

    for n in (1, 4, 8, 16, 32):
        print(f"copy pipeline n={n:2d}  {timeit(lambda: pipe(n)):7.3f} ms")
