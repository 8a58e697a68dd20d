"""Small launches of every product kernel for the bounds-checked build
(tests/test_gpu_bounds.py: the library built with -DSVDLUT_BOUNDS_CHECK traps
on any out-of-range table / slot / accumulator index; compute-sanitizer is
closed on the GPU pool):

    SVDLUT_LIB=paper_2508_16121_b200/_lib/variants/libchecked.so python tools/sanitize_run.py

fused_fwd_kernel (mbarrier slot ring, TMA table staging, texture planes) in
f32, u8 and the L2-loss epilogue over a 2-image batch with a partial last
chunk; pack_kernel from planes and from factors; fused_bwd_kernel (shared
fixed-point scatter, outlier slow path) and its finalize / reconstruct
kernels; the exact kernel.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import __graft_entry__

    __graft_entry__.build_library()
    from paper_2508_16121_b200 import device, synth

    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    for (h, w, dt, ds) in ((37, 260, 33, 17), (21, 131, 17, 8)):
        case = synth.make_batch([0, 1], h=h, w=w, d_t=dt, d_s=ds)
        rgb = case.rgb.copy()  # index edge cases: exact 0 / 1, out of range, non-finite
        special = np.array([0.0, 1.0, -5.0, 5.0, np.nan, np.inf, -np.inf, 1.0 - 2.0 ** -24], np.float32)
        mask = np.random.default_rng(h).random(rgb.shape) < 0.05
        rgb[mask] = np.random.default_rng(w).choice(special, int(mask.sum()))
        case.rgb = rgb
        p = {k: T(getattr(case, k)) for k in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
        planes = device.reconstruct(p["u"], p["s"], p["vt"])
        tables = device.pack_tables(planes, p["lw"], p["lb"], p["grid_planes"], p["gw"], p["gb"])
        tables_f = device.pack_tables_factors(p["u"], p["s"], p["vt"], p["lw"], p["lb"], p["grid_planes"],
                                              p["gw"], p["gb"])
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        y = device.apply(p["rgb"], tables, nonfinite=flag)
        device.apply(p["rgb"][:, :, 3:], tables_f, y0=3, h_total=h)
        u8 = (p["rgb"].clamp(0, 1) * 255).round().to(torch.uint8).permute(0, 2, 3, 1).contiguous()
        device.apply_io(u8, tables, "u8", "u8")
        gy, loss, gmax = device.apply_l2(p["rgb"], p["rgb"].clamp_min(0) ** 0.8, tables)
        device.fused_backward(p["rgb"], gy, planes, p["lw"], p["grid_planes"], p["gw"], tables=tables,
                              gmax=gmax, gsumsq=loss * (2.0 / p["rgb"].numel()) ** 2)
        tgt = p["rgb"].clamp_min(0) ** 0.8
        tgt.view(-1)[:: max(1, tgt.numel() // 7)] += 100.0  # outliers: the f32 slow path
        device.fused_l2_step(p["rgb"], tgt, tables, planes, p["lw"], p["grid_planes"], p["gw"])
        g = device.fused_backward(p["rgb"], torch.randn_like(y), planes, p["lw"], p["grid_planes"], p["gw"])
        device.reconstruct_backward(p["u"], p["s"], p["vt"], g["dlut_planes"])
        device.apply_exact(p["rgb"], planes, p["lw"], p["lb"], p["grid_planes"], p["gw"], p["gb"])
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
