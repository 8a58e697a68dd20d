"""Reference-facing operator: ``fused_enhance`` on host (numpy) values.

Mirrors ``svdlut.transform.fused_enhance`` (reference transform.py:308-353):
same signature, same validation order and exception classes, exactly one
output raster allocated through ``_alloc_raster`` (observable through
``_raster_hook``, reference transform.py:50-58), and a new ``Image`` returned.

The work runs on the GPU through ``svdlut_enhance_host`` (C ABI): the image
and tables are copied host→device, the tables are packed on device, the fused
sm_100a kernel runs, and the result is copied back — pipelined over row
strips on two streams.  ``threads`` is accepted for signature compatibility
and ignored.  The output raster is page-locked so the device→host copy is a
direct DMA.  There is no CPU path: without the built library or a GPU this
raises.
"""

import atexit
import ctypes
import threading

import numpy as np

from . import _lib
from .core_types import Image as _Image
from .errors import BadGridCount, CudaError, DegenerateImage, DimensionMismatch, NonFiniteValue

__all__ = ["fused_enhance", "enhance_payload", "naive_enhance", "slice_grid2d", "apply_lut2d",
           "combine_slices", "apply_lut3d", "_alloc_raster"]

# Test instrumentation: called with the shape of every raster this module
# allocates (the reference's contract; transform.py:50-58).
_raster_hook = None


def _alloc_raster(shape):
    if _raster_hook is not None:
        _raster_hook(shape)
    return _pinned_empty(shape)


def _pinned_payload(shape, fmt):
    """Page-locked output payload (uint8 or big-endian uint16) so the D2H
    copies run at full PCIe rate; pageable memory if pinning is unavailable."""
    try:
        import torch

        n = int(np.prod(shape)) * (1 if fmt == 1 else 2)
        raw = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
        return raw.view(np.uint8 if fmt == 1 else np.dtype(">u2")).reshape(shape)
    except Exception:  # noqa: BLE001 - pinning is an optimisation only
        return np.empty(shape, np.uint8 if fmt == 1 else np.dtype(">u2"))


def _pinned_empty(shape):
    import torch

    if torch.cuda.is_available():
        return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
    return np.empty(shape, dtype=np.float32)


_ctx_lock = threading.Lock()
_ctxs = {}


def _host_ctx(device):
    with _ctx_lock:
        ctx = _ctxs.get(device)
        if ctx is None:
            ctx = _lib.load().svdlut_ctx_create(device)
            if not ctx:
                raise CudaError(f"could not create a CUDA context on device {device}")
            _ctxs[device] = ctx
        return ctx


@atexit.register
def _release():
    if _lib._lib is None:
        return
    for ctx in _ctxs.values():
        _lib._lib.svdlut_ctx_destroy(ctx)
    _ctxs.clear()


def _current_device():
    import torch

    if not torch.cuda.is_available():
        raise CudaError("no CUDA device: the apply path has no CPU fallback")
    return torch.cuda.current_device()


def _image_type(img):
    """Return an Image class compatible with the caller's (reference or ours)."""
    return type(img)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def fused_enhance(img, luts, lut_weights, grids, grid_weights, threads: int = 1,
                  exact: bool = False, alloc=None):
    """Single-pass LUT transform plus grid slicing on the GPU.

    ``exact=True`` selects the f64 kernel whose output is bitwise equal to the
    reference; the default fp32 kernel agrees within 1e-5 with identical cell
    selection.  ``alloc`` overrides the raster allocator (the plugin passes
    the reference module's ``_alloc_raster`` so its ``_raster_hook`` fires).
    """
    del threads  # the GPU decides its own parallelism
    if grids.k % 3 != 0:
        raise BadGridCount(f"grid count {grids.k} is not a multiple of 3")
    if grid_weights.k != grids.k:
        raise DimensionMismatch(f"{grids.k} grids but {grid_weights.k} weight rows")
    if img.width < 2 or img.height < 2:
        raise DegenerateImage("slicing needs at least 2 px in each direction")
    h, w = img.height, img.width
    out = (alloc or _alloc_raster)((3, h, w))
    if not (out.flags.c_contiguous and out.dtype == np.float32 and out.flags.writeable):
        raise DimensionMismatch("raster allocator must return a writable float32 C-contiguous array")
    rgb = _c32(img.data)
    planes = _c32(luts.planes)
    lw, lb = _c32(lut_weights.w), _c32(lut_weights.b)
    gp = _c32(grids.planes)
    gw, gb = _c32(grid_weights.w), _c32(grid_weights.b)
    flag = ctypes.c_int(0)
    ctx = _host_ctx(_current_device())
    _lib.call("svdlut_enhance_host", ctx, _ptr(rgb), h, w, _ptr(planes), _ptr(lw), _ptr(lb),
              planes.shape[2], _ptr(gp), _ptr(gw), _ptr(gb), gp.shape[0], gp.shape[2], _ptr(out),
              int(bool(exact)), ctypes.byref(flag))
    cls = _image_type(img)
    # the non-finite flag is only produced by the fast kernel; the exact kernel
    # also serves dims beyond shared memory (svdlut_fast_supported)
    fast = not exact and bool(_lib.load().svdlut_fast_supported(planes.shape[2], gp.shape[2]))
    if fast and issubclass(cls, _Image):
        if flag.value:
            raise NonFiniteValue("image data contains a NaN or infinite entry")
        return cls._trusted(w, h, out)
    return cls(w, h, out)  # exact kernel / foreign Image type: the constructor validates


def enhance_payload(payload, luts, lut_weights, grids, grid_weights, out_bits=None, out=None):
    """pnm.load -> fused_enhance -> pnm.save's payload, fused on the GPU.

    ``payload``: a PNM P6 sample array (H, W, 3), uint8 (maxval 255) or
    big-endian uint16 ``'>u2'`` (maxval 65535) — what reference pnm.py reads
    and writes after the header.  Samples decode as f32(f64(v) / maxval)
    (pnm.py:79), the fast fp32 apply runs, and the result is quantized as
    floor(clip(y, 0, 1) * maxval + 0.5) (pnm.py:83-86) in the kernel epilogue;
    only 6 (u8) or 12 (u16) bytes per pixel cross PCIe.  ``out_bits`` (8 or
    16) defaults to the input's; ``out`` (optional) receives the result
    (page-locked memory keeps the copies at full PCIe rate).  Against the reference chain the result
    differs only where the fp32 output (within 1e-5 of the reference) falls on
    the other side of a quantization boundary (±1).
    """
    pl = np.asarray(payload)
    if pl.ndim != 3 or pl.shape[2] != 3:
        raise DimensionMismatch(f"payload must be (H, W, 3), got {pl.shape}")
    if pl.dtype == np.uint8:
        fi, in_bits = 1, 8
    elif pl.dtype in (np.dtype(">u2"), np.dtype("<u2")):
        fi, in_bits = 2, 16
        pl = pl.astype(">u2", copy=False)
    else:
        raise DimensionMismatch(f"payload dtype must be uint8 or >u2, got {pl.dtype}")
    out_bits = in_bits if out_bits is None else out_bits
    if out_bits not in (8, 16):
        raise DimensionMismatch(f"out_bits must be 8 or 16, got {out_bits}")
    if grids.k % 3 != 0:
        raise BadGridCount(f"grid count {grids.k} is not a multiple of 3")
    if grid_weights.k != grids.k:
        raise DimensionMismatch(f"{grids.k} grids but {grid_weights.k} weight rows")
    h, w = pl.shape[0], pl.shape[1]
    if w < 2 or h < 2:
        raise DegenerateImage("slicing needs at least 2 px in each direction")
    pl = np.ascontiguousarray(pl)
    fo = 1 if out_bits == 8 else 2
    odt = np.dtype(np.uint8) if fo == 1 else np.dtype(">u2")
    if out is None:
        out = _pinned_payload((h, w, 3), fo)
    elif out.shape != (h, w, 3) or out.dtype != odt or not out.flags.c_contiguous:
        raise DimensionMismatch(f"out must be a C-contiguous (H, W, 3) {odt} array")
    planes = _c32(luts.planes)
    lw, lb = _c32(lut_weights.w), _c32(lut_weights.b)
    gp = _c32(grids.planes)
    gw, gb = _c32(grid_weights.w), _c32(grid_weights.b)
    flag = ctypes.c_int(0)
    ctx = _host_ctx(_current_device())
    _lib.call("svdlut_enhance_host_io", ctx, _ptr(pl), fi, h, w, _ptr(planes), _ptr(lw), _ptr(lb),
              planes.shape[2], _ptr(gp), _ptr(gw), _ptr(gb), gp.shape[0], gp.shape[2], _ptr(out), fo,
              ctypes.byref(flag))
    if flag.value:
        raise NonFiniteValue("enhanced image contains a NaN or infinite entry")
    return out


# ---- multi-pass "original structure" and the 3D-LUT baseline ---------------------
# Reference transform.py:93-212 on the GPU (svdlut_naive.cu): every stage is an
# f64 kernel with the reference's numpy operation order and f32 rasters
# between stages, so results are bitwise equal to the reference.  They exist
# for the multi-stage vs fused comparison; the product path is fused_enhance.

def _to_dev(a):
    import torch

    a = np.ascontiguousarray(a, dtype=np.float32)
    if not a.flags.writeable:  # frozen value types: torch wants a writable buffer
        a = a.copy()
    return torch.from_numpy(a).to(torch.device("cuda", _current_device()))


def _to_host_raster(t, shape, alloc=None):
    out = (alloc or _alloc_raster)(shape)
    out[...] = t.cpu().numpy().reshape(shape)
    return out


def slice_grid2d(img, grids, weights, alloc=None):
    """(K, H, W) slicing maps of every grid (transform.py:152-178)."""
    from . import device
    from .core_types import SpatialFeatureMap

    if img.width < 2 or img.height < 2:
        raise DegenerateImage("slicing needs at least 2 px in each direction")
    if weights.k != grids.k:
        raise DimensionMismatch(f"{grids.k} grids but {weights.k} weight rows")
    fs = device.slice_grids(_to_dev(img.data)[None], _to_dev(grids.planes)[None],
                            _to_dev(weights.w)[None], _to_dev(weights.b)[None])
    return SpatialFeatureMap(_to_host_raster(fs[0], (grids.k, img.height, img.width), alloc))


def apply_lut2d(img, luts, weights, alloc=None):
    """Weighted 2D-LUT transform + channel bias (transform.py:123-141)."""
    from . import device

    y = device.apply_lut2d(_to_dev(img.data)[None], _to_dev(luts.planes)[None],
                           _to_dev(weights.w)[None], _to_dev(weights.b)[None])
    return _image_type(img)(img.width, img.height,
                            _to_host_raster(y[0], (3, img.height, img.width), alloc))


def combine_slices(base, fs, alloc=None):
    """base + sum of the maps j = c, c+3, ... onto channel c (transform.py:181-193)."""
    from . import device

    if fs.k % 3 != 0:
        raise BadGridCount(f"grid count {fs.k} is not a multiple of 3")
    if tuple(fs.data.shape[1:]) != (base.height, base.width):
        raise DimensionMismatch("feature map size differs from image size")
    y = device.combine_slices(_to_dev(base.data)[None], _to_dev(fs.data)[None])
    return _image_type(base)(base.width, base.height,
                             _to_host_raster(y[0], (3, base.height, base.width), alloc))


def naive_enhance(img, luts, lut_weights, grids, grid_weights, alloc=None):
    """Slice, transform, then combine (transform.py:196-212): the multi-stage
    composition with every intermediate raster materialized — like the
    reference, each stage allocates its raster through ``_alloc_raster``
    ((K, H, W), then two (3, H, W)), so the raster hook sees the same pattern."""
    if grids.k % 3 != 0:
        raise BadGridCount(f"grid count {grids.k} is not a multiple of 3")
    fs = slice_grid2d(img, grids, grid_weights, alloc=alloc)
    base = apply_lut2d(img, luts, lut_weights, alloc=alloc)
    return combine_slices(base, fs, alloc=alloc)


def apply_lut3d(img, lut, alloc=None):
    """Trilinear 3D LUT transform, one cube per output channel (transform.py:93-120)."""
    from . import device

    y = device.apply_lut3d(_to_dev(img.data)[None], _to_dev(lut.tables)[None])
    return _image_type(img)(img.width, img.height,
                            _to_host_raster(y[0], (3, img.height, img.width), alloc))
