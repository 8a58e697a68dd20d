"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool).

* The library rebuilt with -DSVDLUT_BOUNDS_CHECK checks every table, texture,
  slot-ring and accumulator index the kernels form and traps on a violation;
  tools/sanitize_run.py drives every product kernel through it (f32 / u8 /
  L2 forward over a batch with partial chunks, row strips, both packers,
  backward with its outlier path, exact kernel) on inputs with exact 0 / 1,
  out-of-range and non-finite samples.
* Guard bands: outputs written into the middle of sentinel-filled buffers
  (every byte around them must survive), inputs bordered by NaN (an
  out-of-bounds read would poison the result, which must equal the
  guard-free run bit for bit).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2508_16121_b200", "_lib", "variants", "libchecked.so")


def _stale(lib):
    import glob

    if not os.path.exists(lib):
        return True
    srcs = glob.glob(os.path.join(ROOT, "paper_2508_16121_b200", "csrc", "*"))
    return any(os.path.getmtime(f) > os.path.getmtime(lib) for f in srcs)


def test_bounds_checked_build_runs_clean():
    if _stale(CHECKED):
        res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), "checked",
                              "-DSVDLUT_BOUNDS_CHECK"], cwd=ROOT, capture_output=True, text=True, timeout=1800)
        assert res.returncode == 0, res.stderr[-3000:]
    env = dict(os.environ, SVDLUT_LIB=CHECKED)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=1800)
    assert res.returncode == 0 and "sanitize_run ok" in res.stdout, (res.stdout + res.stderr)[-3000:]


def _guarded(shape, dtype, fill, dev):
    import torch

    n = int(np.prod(shape))
    pad = 4096
    buf = torch.full((n + 2 * pad,), fill, dtype=dtype, device=dev)
    return buf, buf[pad:pad + n].view(*shape), pad


def test_guard_bands_forward_and_backward():
    import torch

    import __graft_entry__

    __graft_entry__.build_library()
    from paper_2508_16121_b200 import device, synth

    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    case = synth.make_batch([3, 4], h=45, w=301)
    p = {k: T(getattr(case, k)) for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    tables = device.pack_tables_factors(*(p[k] for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")))
    shape = case.rgb.shape
    xbuf, x, _ = _guarded(shape, torch.float32, float("nan"), dev)
    x.copy_(T(case.rgb))
    want = device.apply(T(case.rgb), tables)
    obuf, out, pad = _guarded(shape, torch.float32, 12345.0, dev)
    device.apply(x, tables, out=out)
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    n = out.numel()
    assert bool((obuf[:pad] == 12345.0).all()) and bool((obuf[pad + n:] == 12345.0).all())
    # u8 payload in / out
    u8 = (T(case.rgb).clamp(0, 1) * 255).round().to(torch.uint8).permute(0, 2, 3, 1).contiguous()
    ubuf, uo, upad = _guarded(u8.shape, torch.uint8, 77, dev)
    device.apply_io(u8, tables, "u8", "u8", out=uo)
    torch.cuda.synchronize()
    assert torch.equal(uo, device.apply_io(u8, tables, "u8", "u8"))
    assert bool((ubuf[:upad] == 77).all()) and bool((ubuf[upad + uo.numel():] == 77).all())
    # backward: gradient image in a guarded buffer, gY bordered by NaN
    planes = device.reconstruct(p["u"], p["s"], p["vt"])
    gyb, gy, _ = _guarded(shape, torch.float32, float("nan"), dev)
    gy.copy_(torch.randn(shape, device=dev))
    ref = device.fused_backward(x.clone(), gy.clone(), planes, p["lw"], p["grid_planes"], p["gw"])
    g = device.fused_backward(x, gy, planes, p["lw"], p["grid_planes"], p["gw"])
    torch.cuda.synchronize()
    for k in ref:
        assert torch.isfinite(g[k]).all(), k
        assert float((g[k] - ref[k]).abs().max()) <= 1e-6 * max(1.0, float(ref[k].abs().max())), k
