"""Duplex probe (development tool): the fused kernel reading its input from
pinned host memory (zero-copy) while a copy engine moves an unrelated 4K
image device -> host, and the mirror case (DMA H2D || kernel writing host
memory).  Tells whether SM-issued PCIe traffic and copy-engine traffic in the
other direction run at full duplex rate."""
import ctypes
import os
import sys

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
pin_other = torch.empty_like(pin_in).pin_memory()
d_in = pin_in.to(dev)
d_out = torch.empty_like(d_in)
d_other = torch.empty_like(d_in)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
sk, sc = torch.cuda.Stream(), torch.cuda.Stream()


def kern(src, dst):
    _lib.call("svdlut_fused_fwd_packed_ex", P(src), 1, H, W, 0, H, P(tables.buf), 33, 17, P(dst),
              None, 0, None, -1, sk.cuda_stream)


def timed(k=None, c=None, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0.record(sk)
        sc.wait_event(e0)
        if k:
            k()
        if c:
            with torch.cuda.stream(sc):
                c()
        sk.wait_stream(sc)
        e1.record(sk)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[n // 2]


d2h = lambda: pin_other.copy_(d_other, non_blocking=True)  # noqa: E731
h2d = lambda: d_other.copy_(pin_other, non_blocking=True)  # noqa: E731
print(f"kernel zc-in alone        {timed(lambda: kern(pin_in, d_out)):.3f} ms")
print(f"D2H copy alone            {timed(c=d2h):.3f} ms")
print(f"kernel zc-in || D2H copy  {timed(lambda: kern(pin_in, d_out), d2h):.3f} ms")
print(f"kernel zc-out alone       {timed(lambda: kern(d_in, pin_out)):.3f} ms")
print(f"H2D copy alone            {timed(c=h2d):.3f} ms")
print(f"kernel zc-out || H2D copy {timed(lambda: kern(d_in, pin_out), h2d):.3f} ms")
