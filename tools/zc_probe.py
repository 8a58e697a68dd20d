"""Zero-copy probe (development tool): the fused kernel reading its input from
and writing its output to pinned host memory directly over PCIe, vs the
device-resident kernel and the staged copies."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build_library()
from paper_2508_16121_b200 import _lib, device, synth  # noqa: E402

H, W = 2160, 3840
dev = torch.device("cuda", 0)
case = synth.make_case(0)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
planes = device.reconstruct(T(case.u), T(case.s), T(case.vt))
tables = device.pack_tables(planes, T(case.lw), T(case.lb), T(case.grid_planes), T(case.gw), T(case.gb))
pin_in = torch.empty((1, 3, H, W), dtype=torch.float32, pin_memory=True)
pin_in.copy_(torch.from_numpy(case.rgb)[None])
pin_out = torch.empty_like(pin_in).pin_memory()
d_in = pin_in.to(dev)
d_out = torch.empty_like(d_in)
P = lambda t: None if t is None else __import__("ctypes").c_void_p(t.data_ptr())  # noqa: E731


def run(src, dst):
    _lib.call("svdlut_fused_fwd_packed_ex", P(src), 1, H, W, 0, H, P(tables.buf), 33, 17, P(dst),
              None, 0, None, -1, torch.cuda.current_stream().cuda_stream)


def timeit(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print(f"device->device   {timeit(lambda: run(d_in, d_out)):7.3f} ms")
print(f"host->device     {timeit(lambda: run(pin_in, d_out)):7.3f} ms")
print(f"device->host     {timeit(lambda: run(d_in, pin_out)):7.3f} ms")
print(f"host->host       {timeit(lambda: run(pin_in, pin_out)):7.3f} ms")
run(d_in, d_out)
run(pin_in, pin_out)
torch.cuda.synchronize()
print("equal:", torch.equal(d_out.cpu(), pin_out))
