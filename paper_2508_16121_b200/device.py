"""Device-tensor API over the C ABI (torch is the allocator and stream source).

Everything here takes CUDA float32 tensors that are already resident in HBM
and launches on ``torch.cuda.current_stream()``; nothing copies to the host.
Shapes (B = batch of independent images, each with its own tables):

    rgb / out      (B, 3, H, W)          planar, C-contiguous
    lut_planes     (B, 3, 3, d_t, d_t)   [out channel][rg|rb|gb][a][b]
    lw, lb         (B, 3, 3), (B, 3)
    grid_planes    (B, K, 3, d_s, d_s)   [grid][xy|xc|yc][a][b]
    gw, gb         (B, K, 3), (B, K)
    u, s, vt       (B, 3, 3, d_t, n), (B, 3, 3, n), (B, 3, 3, n, d_t)

Unbatched inputs (no leading B) are accepted and promoted to B = 1.
(y0, h_total) evaluate a row strip of a taller image (global normalisation).
"""

import ctypes

import torch

from . import _lib
from .errors import DimensionMismatch

__all__ = [
    "apply_io", "FMT_F32", "FMT_U8", "FMT_U16BE", "apply_l2",
    "table_bytes", "fast_supported", "PackedTables", "reconstruct", "pack_tables",
    "pack_tables_factors", "apply",
    "apply_exact", "slice_grids", "apply_lut2d", "combine_slices", "apply_lut3d",
    "fused_forward", "indices", "fused_backward", "fused_l2_step", "reconstruct_backward",
]


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(t):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _call(t, name, *args):
    """C-ABI call with t's device current (the library launches on, and
    creates texture objects for, the current device)."""
    with torch.cuda.device(t.device):
        _lib.call(name, *args)


def _f32(t, name, ndim):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != torch.float32:
        raise DimensionMismatch(f"{name} must be float32, got {t.dtype}")
    if not t.is_cuda:
        raise DimensionMismatch(f"{name} must be a CUDA tensor")
    if t.dim() == ndim - 1:
        t = t.unsqueeze(0)
    if t.dim() != ndim:
        raise DimensionMismatch(f"{name} must have {ndim} dims (batched), got {tuple(t.shape)}")
    return t.contiguous()


def table_bytes(d_t, d_s):
    return int(_lib.load().svdlut_table_bytes(d_t, d_s))


def fast_supported(d_t, d_s):
    return bool(_lib.load().svdlut_fast_supported(d_t, d_s))


class PackedTables:
    """Per-image coefficient tables produced by the on-device prologue."""

    def __init__(self, buf, batch, d_t, d_s):
        self.buf, self.batch, self.d_t, self.d_s = buf, batch, d_t, d_s

    @property
    def device(self):
        return self.buf.device


def reconstruct(u, s, vt):
    """svd.reconstruct_lut on device: planes = f32((f64 u * f64 s) @ f64 vt)."""
    u, s, vt = _f32(u, "u", 5), _f32(s, "s", 4), _f32(vt, "vt", 5)
    b, _, _, d, n = u.shape
    if tuple(s.shape) != (b, 3, 3, n) or tuple(vt.shape) != (b, 3, 3, n, d):
        raise DimensionMismatch(f"inconsistent factor shapes {tuple(u.shape)} {tuple(s.shape)} "
                                f"{tuple(vt.shape)}")
    planes = torch.empty((b, 3, 3, d, d), dtype=torch.float32, device=u.device)
    _call(u, "svdlut_reconstruct", _p(u), _p(s), _p(vt), b, d, n, _p(planes), _stream(u))
    return planes


def _check_tables(lut_planes, lw, lb, grid_planes, gw, gb):
    lp = _f32(lut_planes, "lut_planes", 5)
    lw, lb = _f32(lw, "lw", 3), _f32(lb, "lb", 2)
    gp = _f32(grid_planes, "grid_planes", 5)
    gw, gb = _f32(gw, "gw", 3), _f32(gb, "gb", 2)
    b, d_t = lp.shape[0], lp.shape[3]
    k, d_s = gp.shape[1], gp.shape[3]
    if tuple(lp.shape[1:3]) != (3, 3) or lp.shape[3] != lp.shape[4]:
        raise DimensionMismatch(f"lut_planes must be (B,3,3,d,d), got {tuple(lp.shape)}")
    if gp.shape[2] != 3 or gp.shape[3] != gp.shape[4]:
        raise DimensionMismatch(f"grid_planes must be (B,K,3,d,d), got {tuple(gp.shape)}")
    if tuple(lw.shape) != (b, 3, 3) or tuple(lb.shape) != (b, 3):
        raise DimensionMismatch("LUT weights must be (B,3,3) and (B,3)")
    if gw.shape[0] != b or gw.shape[2] != 3 or gb.shape[0] != b or gp.shape[0] != b:
        raise DimensionMismatch("grid tensors disagree on the batch size")
    if gw.shape[1] != k or gb.shape[1] != k:
        raise DimensionMismatch(f"{k} grids but {gw.shape[1]} weight rows")
    return lp, lw, lb, gp, gw, gb, b, d_t, k, d_s


def pack_tables(lut_planes, lw, lb, grid_planes, gw, gb):
    """Fold weights, merge grids per channel, write coefficient cells."""
    lp, lw, lb, gp, gw, gb, b, d_t, k, d_s = _check_tables(lut_planes, lw, lb, grid_planes, gw, gb)
    nbytes = table_bytes(d_t, d_s)
    buf = torch.empty(b * nbytes // 4, dtype=torch.float32, device=lp.device)
    _call(lp, "svdlut_pack_tables", _p(lp), _p(lw), _p(lb), d_t, _p(gp), _p(gw), _p(gb), k, d_s,
              b, _p(buf), _stream(lp))
    return PackedTables(buf, b, d_t, d_s)


def pack_tables_factors(u, s, vt, lw, lb, grid_planes, gw, gb):
    """Tables straight from the SVD factors (reconstruct fused into packing)."""
    u, s, vt = _f32(u, "u", 5), _f32(s, "s", 4), _f32(vt, "vt", 5)
    b, _, _, d, n = u.shape
    if tuple(s.shape) != (b, 3, 3, n) or tuple(vt.shape) != (b, 3, 3, n, d):
        raise DimensionMismatch(f"inconsistent factor shapes {tuple(u.shape)} {tuple(s.shape)} "
                                f"{tuple(vt.shape)}")
    lw, lb = _f32(lw, "lw", 3), _f32(lb, "lb", 2)
    gp = _f32(grid_planes, "grid_planes", 5)
    gw, gb = _f32(gw, "gw", 3), _f32(gb, "gb", 2)
    k, d_s = gp.shape[1], gp.shape[3]
    if tuple(lw.shape) != (b, 3, 3) or tuple(lb.shape) != (b, 3) or gp.shape[0] != b:
        raise DimensionMismatch("weights / grids disagree with the factors' batch")
    if tuple(gw.shape) != (b, k, 3) or tuple(gb.shape) != (b, k):
        raise DimensionMismatch(f"{k} grids but weights shaped {tuple(gw.shape)} {tuple(gb.shape)}")
    nbytes = table_bytes(d, d_s)
    buf = torch.empty(b * nbytes // 4, dtype=torch.float32, device=u.device)
    _call(u, "svdlut_pack_tables_factors", _p(u), _p(s), _p(vt), n, _p(lw), _p(lb), d, _p(gp),
              _p(gw), _p(gb), k, d_s, b, _p(buf), _stream(u))
    return PackedTables(buf, b, d, d_s)


def _image(rgb, batch):
    rgb = _f32(rgb, "rgb", 4)
    if rgb.shape[1] != 3:
        raise DimensionMismatch(f"rgb must be (B,3,H,W), got {tuple(rgb.shape)}")
    if batch is not None and rgb.shape[0] != batch:
        raise DimensionMismatch(f"{rgb.shape[0]} images but tables for {batch}")
    return rgb


def apply(rgb, tables, out=None, y0=0, h_total=None, nonfinite=None):
    """Fused slice + LUT apply (fast fp32 kernel) from packed tables.

    ``nonfinite``: optional int32 CUDA tensor (1 element) OR-ed with 1 if any
    output is NaN/Inf.  One kernel launch.
    """
    rgb = _image(rgb, tables.batch)
    b, _, h, w = rgb.shape
    h_total = h if h_total is None else h_total
    if out is None:
        out = torch.empty_like(rgb)
    elif out.shape != rgb.shape or not out.is_contiguous() or out.dtype != torch.float32:
        raise DimensionMismatch("out must be a contiguous float32 tensor shaped like rgb")
    _call(rgb, "svdlut_fused_fwd_packed_ex", _p(rgb), b, h, w, y0, h_total, _p(tables.buf),
              tables.d_t, tables.d_s, _p(out), _p(None), 0, _p(nonfinite), _stream(rgb))
    return out


FMT_F32, FMT_U8, FMT_U16BE = 0, 1, 2  # include/svdlut_b200.h SVDLUT_FMT_*
_FMT_NAMES = {"f32": FMT_F32, "u8": FMT_U8, "u16be": FMT_U16BE}


def _fmt(f):
    return _FMT_NAMES[f] if isinstance(f, str) else int(f)


def _io_image(t, fmt, batch):
    """(B, H, W) of an image tensor in sample format fmt: f32 (B,3,H,W);
    u8 (B,H,W,3) uint8; u16be (B,H,W,6) uint8 = 3 big-endian samples."""
    if fmt == FMT_F32:
        t = _image(t, batch)
        return t, t.shape[0], t.shape[2], t.shape[3]
    if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8 or not t.is_cuda:
        raise DimensionMismatch("integer images must be CUDA uint8 tensors")
    last = 3 if fmt == FMT_U8 else 6
    if t.dim() == 3:
        t = t.unsqueeze(0)
    if t.dim() != 4 or t.shape[3] != last or not t.is_contiguous():
        raise DimensionMismatch(f"expected a contiguous (B, H, W, {last}) uint8 image, got {tuple(t.shape)}")
    if batch is not None and t.shape[0] != batch:
        raise DimensionMismatch(f"{t.shape[0]} images but tables for {batch}")
    return t, t.shape[0], t.shape[1], t.shape[2]


def apply_io(x, tables, in_fmt="f32", out_fmt="f32", out=None, y0=0, h_total=None, nonfinite=None):
    """Fused apply with PNM sample formats on either side: integer input is
    decoded as pnm.load does (f32(f64(v) / maxval), pnm.py:79), integer
    output quantized as pnm.save does (floor(clip(y,0,1)*maxval + 0.5),
    pnm.py:83-86) — inside the kernel, so u8 in/out moves 6 B/pixel instead
    of 24.  Formats: "f32" (B,3,H,W) float32, "u8" (B,H,W,3) uint8, "u16be"
    (B,H,W,6) uint8 holding big-endian uint16 samples."""
    fi, fo = _fmt(in_fmt), _fmt(out_fmt)
    x, b, h, w = _io_image(x, fi, tables.batch)
    h_total = h if h_total is None else h_total
    if out is None:
        if fo == FMT_F32:
            out = torch.empty((b, 3, h, w), dtype=torch.float32, device=x.device)
        else:
            out = torch.empty((b, h, w, 3 if fo == FMT_U8 else 6), dtype=torch.uint8, device=x.device)
    else:
        out, bo, ho, wo = _io_image(out, fo, tables.batch)
        if (bo, ho, wo) != (b, h, w):
            raise DimensionMismatch("out does not match the input image size")
    _call(x, "svdlut_fused_fwd_io", _p(x), fi, b, h, w, y0, h_total, _p(tables.buf), tables.d_t,
              tables.d_s, _p(out), fo, _p(nonfinite), _stream(x))
    return out


# ---- multi-pass "original structure" and the 3D-LUT baseline (f64 stages,
#      bitwise equal to the reference's numpy; svdlut_naive.cu) -------------------
def slice_grids(rgb, grid_planes, gw, gb, y0=0, h_total=None):
    """(B, K, H, W) slicing maps (reference transform.slice_grid2d)."""
    gp, gw, gb = _f32(grid_planes, "grid_planes", 5), _f32(gw, "gw", 3), _f32(gb, "gb", 2)
    rgb = _image(rgb, gp.shape[0])
    b, _, h, w = rgb.shape
    k, d_s = gp.shape[1], gp.shape[3]
    if gw.shape[1] != k or gb.shape[1] != k:
        raise DimensionMismatch(f"{k} grids but {gw.shape[1]} weight rows")
    fs = torch.empty((b, k, h, w), dtype=torch.float32, device=rgb.device)
    _call(rgb, "svdlut_slice_grids", _p(rgb), b, h, w, y0, h if h_total is None else h_total, _p(gp),
              _p(gw), _p(gb), k, d_s, _p(fs), _stream(rgb))
    return fs


def apply_lut2d(rgb, lut_planes, lw, lb):
    """(B, 3, H, W) weighted 2D-LUT transform (reference transform.apply_lut2d)."""
    lp, lw, lb = _f32(lut_planes, "lut_planes", 5), _f32(lw, "lw", 3), _f32(lb, "lb", 2)
    rgb = _image(rgb, lp.shape[0])
    b, _, h, w = rgb.shape
    out = torch.empty_like(rgb)
    _call(rgb, "svdlut_apply_lut2d", _p(rgb), b, h, w, _p(lp), _p(lw), _p(lb), lp.shape[3], _p(out),
              _stream(rgb))
    return out


def combine_slices(base, fs):
    """base + channel-grouped slicing maps (reference transform.combine_slices)."""
    base = _image(base, None)
    fs = _f32(fs, "fs", 4)
    if fs.shape[0] != base.shape[0] or fs.shape[2:] != base.shape[2:]:
        raise DimensionMismatch("feature map size differs from image size")
    b, _, h, w = base.shape
    out = torch.empty_like(base)
    _call(base, "svdlut_combine_slices", _p(base), _p(fs), b, h, w, fs.shape[1], _p(out),
              _stream(base))
    return out


def apply_lut3d(rgb, cubes):
    """(B, 3, H, W) trilinear 3D LUT, cubes (B, 3, d, d, d) (reference apply_lut3d)."""
    cubes = _f32(cubes, "cubes", 5)
    rgb = _image(rgb, cubes.shape[0])
    b, _, h, w = rgb.shape
    out = torch.empty_like(rgb)
    _call(rgb, "svdlut_apply_lut3d", _p(rgb), b, h, w, _p(cubes), cubes.shape[2], _p(out),
              _stream(rgb))
    return out


def apply_exact(rgb, lut_planes, lw, lb, grid_planes, gw, gb, out=None, y0=0, h_total=None):
    """f64 op-for-op kernel: bitwise equal to the reference fused_enhance."""
    lp, lw, lb, gp, gw, gb, bt, d_t, k, d_s = _check_tables(lut_planes, lw, lb, grid_planes, gw, gb)
    rgb = _image(rgb, bt)
    b, _, h, w = rgb.shape
    h_total = h if h_total is None else h_total
    if out is None:
        out = torch.empty_like(rgb)
    _call(rgb, "svdlut_fused_fwd_exact", _p(rgb), b, h, w, y0, h_total, _p(lp), _p(lw), _p(lb), d_t,
              _p(gp), _p(gw), _p(gb), k, d_s, _p(out), _stream(rgb))
    return out


def fused_forward(rgb, lut_planes, lw, lb, grid_planes, gw, gb, out=None, y0=0, h_total=None,
                  exact=False):
    """Pack + apply; dimensions beyond the shared-memory kernel use the exact kernel."""
    if exact or not fast_supported(lut_planes.shape[-1], grid_planes.shape[-1]):
        return apply_exact(rgb, lut_planes, lw, lb, grid_planes, gw, gb, out, y0, h_total)
    tables = pack_tables(lut_planes, lw, lb, grid_planes, gw, gb)
    return apply(rgb, tables, out=out, y0=y0, h_total=h_total)


def indices(rgb, d_t, d_s, y0=0, h_total=None):
    """(B, 8, H, W) int32 cell selection as the fast kernel computes it."""
    rgb = _image(rgb, None)
    b, _, h, w = rgb.shape
    h_total = h if h_total is None else h_total
    idx = torch.empty((b, 8, h, w), dtype=torch.int32, device=rgb.device)
    _call(rgb, "svdlut_indices", _p(rgb), b, h, w, y0, h_total, d_t, d_s, _p(idx), _stream(rgb))
    return idx


def apply_l2(rgb, target, tables, gscale=None, y0=0, h_total=None):
    """Training-step forward with the L2 loss fused into the epilogue.

    Returns (gy, loss_sum, gmax): gy = (Y - target) * gscale (default 2/N,
    i.e. d mean((Y-T)^2)/dY), loss_sum (B,) float64 = per-image sum of squared
    residuals, gmax (B,) = per-image max |gy| (feeds fused_backward's
    fixed-point scale).  Y itself is never written to HBM.
    """
    rgb = _image(rgb, tables.batch)
    target = _image(target, tables.batch)
    if target.shape != rgb.shape:
        raise DimensionMismatch("target must be shaped like rgb")
    b, _, h, w = rgb.shape
    gscale = 2.0 / rgb.numel() if gscale is None else float(gscale)
    gy = torch.empty_like(rgb)
    loss = torch.empty(b, dtype=torch.float64, device=rgb.device)
    gmax = torch.empty(b, dtype=torch.float32, device=rgb.device)
    _call(rgb, "svdlut_fused_fwd_l2", _p(rgb), _p(target), b, h, w, y0, h if h_total is None else h_total,
              _p(tables.buf), tables.d_t, tables.d_s, _p(gy), _p(loss), _p(gmax),
              ctypes.c_float(gscale), _stream(rgb))
    return gy, loss, gmax


def fused_backward(rgb, gy, lut_planes, lw, grid_planes, gw, y0=0, h_total=None, need_gx=True,
                   tables=None, gmax=None, gsumsq=None):
    """Gradients of the fused apply w.r.t. the input and every table.

    ``tables`` (the forward's PackedTables) and ``gmax`` / ``gsumsq``
    (per-image max |gy| and float64 sum of gy^2, e.g. from apply_l2) skip the
    backward's own table packing and statistics pass.  Returns dict(gx,
    dlut_planes, dlw, dlb, dgrid_planes, dgw, dgb).
    """
    lp = _f32(lut_planes, "lut_planes", 5)
    lw = _f32(lw, "lw", 3)
    gp = _f32(grid_planes, "grid_planes", 5)
    gw = _f32(gw, "gw", 3)
    b, d_t = lp.shape[0], lp.shape[3]
    k, d_s = gp.shape[1], gp.shape[3]
    rgb = _image(rgb, b)
    gy = _image(gy, b)
    if gy.shape != rgb.shape:
        raise DimensionMismatch("gy must be shaped like rgb")
    _, _, h, w = rgb.shape
    h_total = h if h_total is None else h_total
    dev = rgb.device
    g = dict(
        gx=torch.empty_like(rgb) if need_gx else None,
        dlut_planes=torch.empty_like(lp),
        dlw=torch.empty((b, 3, 3), dtype=torch.float32, device=dev),
        dlb=torch.empty((b, 3), dtype=torch.float32, device=dev),
        dgrid_planes=torch.empty_like(gp),
        dgw=torch.empty((b, k, 3), dtype=torch.float32, device=dev),
        dgb=torch.empty((b, k), dtype=torch.float32, device=dev),
    )
    ws_bytes = int(_lib.load().svdlut_bwd_workspace_bytes(b, h, w, d_t, d_s, k))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    if gmax is not None and (gmax.dtype != torch.float32 or gmax.numel() != b):
        raise DimensionMismatch("gmax must be a float32 tensor with one entry per image")
    if gsumsq is not None and (gsumsq.dtype != torch.float64 or gsumsq.numel() != b or gmax is None):
        raise DimensionMismatch("gsumsq must be a float64 tensor with one entry per image (with gmax)")
    _call(rgb, "svdlut_fused_bwd_packed", _p(rgb), _p(gy), b, h, w, y0, h_total,
              _p(tables.buf if tables is not None else None), _p(gmax), _p(gsumsq), _p(lp), _p(lw), d_t,
              _p(gp), _p(gw), k, d_s, _p(g["gx"]), _p(g["dlut_planes"]), _p(g["dlw"]),
              _p(g["dlb"]), _p(g["dgrid_planes"]), _p(g["dgw"]), _p(g["dgb"]), _p(ws), ws_bytes,
              _stream(rgb))
    return g


def fused_l2_step(rgb, target, tables, lut_planes, lw, grid_planes, gw, gscale=None, y0=0, h_total=None,
                  need_gx=True):
    """One pass of the training step's pixel work: Y from ``tables`` (the
    forward's PackedTables), gy = gscale (Y - target) (default 2/N, i.e.
    d mean((Y-T)^2)/dY), and the backward of fused_backward — without gy or Y
    touching HBM.  Returns (loss_sum (B,) float64 per-image sum of squared
    residuals, dict(gx, dlut_planes, dlw, dlb, dgrid_planes, dgw, dgb)).
    """
    lp = _f32(lut_planes, "lut_planes", 5)
    lw = _f32(lw, "lw", 3)
    gp = _f32(grid_planes, "grid_planes", 5)
    gw = _f32(gw, "gw", 3)
    b, d_t = lp.shape[0], lp.shape[3]
    k, d_s = gp.shape[1], gp.shape[3]
    rgb = _image(rgb, b)
    target = _image(target, b)
    if target.shape != rgb.shape:
        raise DimensionMismatch("target must be shaped like rgb")
    if tables.batch != b or tables.d_t != d_t or tables.d_s != d_s:
        raise DimensionMismatch("tables do not match the LUT / grid planes")
    _, _, h, w = rgb.shape
    h_total = h if h_total is None else h_total
    gscale = 2.0 / rgb.numel() if gscale is None else float(gscale)
    dev = rgb.device
    g = dict(
        gx=torch.empty_like(rgb) if need_gx else None,
        dlut_planes=torch.empty_like(lp),
        dlw=torch.empty((b, 3, 3), dtype=torch.float32, device=dev),
        dlb=torch.empty((b, 3), dtype=torch.float32, device=dev),
        dgrid_planes=torch.empty_like(gp),
        dgw=torch.empty((b, k, 3), dtype=torch.float32, device=dev),
        dgb=torch.empty((b, k), dtype=torch.float32, device=dev),
    )
    loss = torch.empty(b, dtype=torch.float64, device=dev)
    ws_bytes = int(_lib.load().svdlut_bwd_workspace_bytes(b, h, w, d_t, d_s, k))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _call(rgb, "svdlut_fused_l2_step", _p(rgb), _p(target), b, h, w, y0, h_total, _p(tables.buf),
          ctypes.c_float(gscale), _p(lp), _p(lw), d_t, _p(gp), _p(gw), k, d_s, _p(g["gx"]),
          _p(g["dlut_planes"]), _p(g["dlw"]), _p(g["dlb"]), _p(g["dgrid_planes"]), _p(g["dgw"]),
          _p(g["dgb"]), _p(loss), _p(ws), ws_bytes, _stream(rgb))
    return loss, g


def reconstruct_backward(u, s, vt, dplanes):
    u, s, vt = _f32(u, "u", 5), _f32(s, "s", 4), _f32(vt, "vt", 5)
    dplanes = _f32(dplanes, "dplanes", 5)
    b, _, _, d, n = u.shape
    du, ds, dvt = torch.empty_like(u), torch.empty_like(s), torch.empty_like(vt)
    _call(u, "svdlut_reconstruct_bwd", _p(u), _p(s), _p(vt), _p(dplanes), b, d, n, _p(du),
              _p(ds), _p(dvt), _stream(u))
    return du, ds, dvt
