"""Pinned-buffer page size vs PCIe copy rate (development tool).

Allocates 25 MB host buffers repeatedly as (a) torch pin_memory and (b)
2 MB-aligned anonymous mmap + madvise(MADV_HUGEPAGE) + cudaHostRegister, and
times one H2D || D2H pair of 6 strips for each (in, out) buffer pair; prints
how much of each buffer the kernel backed with transparent huge pages."""
import ctypes
import mmap
import sys

import numpy as np
import torch

dev = torch.device("cuda", 0)
N = 2160 * 3840 * 3
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), file=sys.stderr)
cudart = torch.cuda.cudart()


def thp_kb(addr, size):
    total = 0
    cur = None
    for line in open("/proc/self/smaps"):
        parts = line.split()
        if "-" in parts[0] and len(parts) > 4:
            lo, hi = (int(x, 16) for x in parts[0].split("-"))
            cur = lo <= addr < hi
        elif cur and parts[0] == "AnonHugePages:":
            total += int(parts[1])
    return total


def huge_buf():
    m = mmap.mmap(-1, N + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    off = (-base) % (2 << 20)
    m.madvise(mmap.MADV_HUGEPAGE, off, N - N % (2 << 20))
    arr = np.frombuffer(m, dtype=np.uint8, count=N, offset=off)
    arr[:] = 1  # fault in
    t = torch.from_numpy(arr)
    rc = cudart.cudaHostRegister(t.data_ptr(), N, 0)
    assert int(rc) == 0, rc
    return t, m


def torch_buf():
    t = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    t.fill_(1)
    return t, None


d_in = torch.empty(N, dtype=torch.uint8, device=dev)
d_out = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def duplex(h_in, h_out, strips=6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record(s1)
        s2.wait_event(e0)
        step = N // strips
        for i in range(strips):
            lo, hi = i * step, N if i == strips - 1 else (i + 1) * step
            with torch.cuda.stream(s1):
                d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
        s1.wait_stream(s2)
        e1.record(s1)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[2]


keep = []
for kind, fn in (("torch", torch_buf), ("huge", huge_buf), ("torch", torch_buf), ("huge", huge_buf),
                 ("torch", torch_buf), ("huge", huge_buf)):
    a, b = fn(), fn()
    keep += [a, b]
    ms = duplex(a[0], b[0])
    print(f"{kind:5s}: duplex {ms:.3f} ms ({2 * N / ms / 1e6:.1f} GB/s)  THP in {thp_kb(a[0].data_ptr(), N) >> 10} MB"
          f" out {thp_kb(b[0].data_ptr(), N) >> 10} MB", file=sys.stderr)
