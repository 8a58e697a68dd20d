"""Copy-engine duplex probe (development tool): pinned host <-> device copies
of one 4K frame (u8 HWC 24.9 MB, f32 planar 99.5 MB) split into strips, H2D on
one stream and D2H on another, both directions at once, 1-D copies."""
import sys

import torch

dev = torch.device("cuda", 0)
for name, nbytes in (("u8", 2160 * 3840 * 3), ("f32", 2160 * 3840 * 12)):
    for strips in (1, 6, 12):
        h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        d_in = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        d_out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        res = {}
        for mode in ("h2d", "d2h", "both"):
            ts = []
            for _ in range(6):
                torch.cuda.synchronize()
                e0.record(s1)
                s2.wait_event(e0)
                step = nbytes // strips
                for i in range(strips):
                    lo, hi = i * step, nbytes if i == strips - 1 else (i + 1) * step
                    if mode in ("h2d", "both"):
                        with torch.cuda.stream(s1):
                            d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
                    if mode in ("d2h", "both"):
                        with torch.cuda.stream(s2):
                            h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
                s1.wait_stream(s2)
                e1.record(s1)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[mode] = sorted(ts)[3]
        gb = nbytes / 1e6
        print(f"{name:4s} strips {strips:2d}: h2d {res['h2d']:.3f} ms ({gb / res['h2d']:.1f} GB/s)  "
              f"d2h {res['d2h']:.3f} ms ({gb / res['d2h']:.1f})  both {res['both']:.3f} ms "
              f"({2 * gb / res['both']:.1f} GB/s total)", file=sys.stderr)
