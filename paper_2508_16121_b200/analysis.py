"""Diagnostics on the GPU (reference analysis.py:1-190).

occurrence_stats counts, per d^3 cube vertex, how often it is a corner of a
pixel's bracketing cell (svdlut_occurrence: shared-memory int32 histograms,
exact u64 totals); utilization_rate derives from the same cube — a vertex of a
pair plane / axis is touched iff the cube's projection / marginal there is
non-zero — so all three modes agree exactly with the reference.  psnr and
delta_e_ab run as float64 reductions on the device (equal to the reference
within floating-point summation order).  Same names, arguments and errors as
the reference.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BadVertexCount, DimensionMismatch

__all__ = ["OccurrenceMap", "utilization_rate", "occurrence_stats", "merge_occurrence", "psnr",
           "delta_e_ab", "heatmap_u16"]

_MODES = ("1d", "2d", "3d")


@dataclass(frozen=True)
class OccurrenceMap:
    """Per-vertex touch counts of a d-vertex cube (analysis.py:34-70)."""

    d: int
    cube: np.ndarray

    def __post_init__(self):
        c = np.ascontiguousarray(self.cube, dtype=np.int64)
        if c.shape != (self.d, self.d, self.d):
            raise DimensionMismatch(f"cube shape {c.shape} does not match d={self.d}")
        if (c < 0).any():
            raise DimensionMismatch("occurrence counts must be nonnegative")
        c.flags.writeable = False
        object.__setattr__(self, "cube", c)

    @property
    def proj_rg(self):
        return self.cube.sum(axis=2)

    @property
    def proj_rb(self):
        return self.cube.sum(axis=1)

    @property
    def proj_gb(self):
        return self.cube.sum(axis=0)

    @property
    def total(self) -> int:
        return int(self.cube.sum())


def _dev_images(images):
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    for img in images:
        a = np.array(img.data, dtype=np.float32, copy=True)
        yield torch.from_numpy(a)[None].to(dev), img.height, img.width


def _count(images, d):
    """u64 cube summed over the images, on the device."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    total = torch.zeros(d ** 3, dtype=torch.int64, device=dev)
    part = torch.empty(d ** 3, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    P = lambda t: __import__("ctypes").c_void_p(t.data_ptr())  # noqa: E731
    for x, h, w in _dev_images(images):
        _lib.call("svdlut_occurrence", P(x), 1, h, w, d, P(part), stream)
        total += part
    return total.reshape(d, d, d).cpu().numpy()


def occurrence_stats(images, d: int) -> OccurrenceMap:
    """Count bracketing-cell corner touches over one or more images."""
    if d < 2:
        raise BadVertexCount(f"need at least 2 vertices, got {d}")
    return OccurrenceMap(d, _count(list(images), d))


def utilization_rate(img, d: int, mode: str = "3d") -> float:
    """Percentage of table vertices touched at least once (analysis.py:74-106)."""
    if d < 2:
        raise BadVertexCount(f"need at least 2 vertices, got {d}")
    mode = mode.lower()
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")
    cube = _count([img], d) > 0
    if mode == "3d":
        return 100.0 * int(cube.sum()) / (d ** 3)
    if mode == "2d":
        touched = int(cube.any(axis=2).sum()) + int(cube.any(axis=1).sum()) + int(cube.any(axis=0).sum())
        return 100.0 * touched / (3 * d * d)
    touched = (int(cube.any(axis=(1, 2)).sum()) + int(cube.any(axis=(0, 2)).sum())
               + int(cube.any(axis=(0, 1)).sum()))
    return 100.0 * touched / (3 * d)


def merge_occurrence(a: OccurrenceMap, b: OccurrenceMap) -> OccurrenceMap:
    if a.d != b.d:
        raise DimensionMismatch(f"cannot merge maps with d={a.d} and d={b.d}")
    return OccurrenceMap(a.d, a.cube + b.cube)


def _pair(a, b):
    if (a.width, a.height) != (b.width, b.height):
        raise DimensionMismatch("images must have equal dimensions")
    (xa, _, _), (xb, _, _) = _dev_images([a, b])
    return xa[0].double(), xb[0].double()


def psnr(a, b) -> float:
    """10*log10(1/MSE), peak 1.0, MSE in float64 (analysis.py:125-137)."""
    xa, xb = _pair(a, b)
    mse = float(((xa - xb) ** 2).mean())
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)


_SRGB_TO_XYZ = np.array([[0.4124564, 0.3575761, 0.1804375],
                         [0.2126729, 0.7151522, 0.0721750],
                         [0.0193339, 0.1191920, 0.9503041]])


def _lab(x):
    import torch

    m = torch.as_tensor(_SRGB_TO_XYZ, dtype=torch.float64, device=x.device)
    rgb = x.clamp(0.0, 1.0)
    lin = torch.where(rgb <= 0.04045, rgb / 12.92, ((rgb + 0.055) / 1.055) ** 2.4)
    xyz = torch.tensordot(m, lin, dims=([1], [0]))
    t = xyz / m.sum(dim=1)[:, None, None]
    delta = 6.0 / 29.0
    f = torch.where(t > delta ** 3, torch.sign(t) * t.abs() ** (1.0 / 3.0),
                    t / (3.0 * delta * delta) + 4.0 / 29.0)
    return torch.stack([116.0 * f[1] - 16.0, 500.0 * (f[0] - f[1]), 200.0 * (f[1] - f[2])])


def delta_e_ab(a, b) -> float:
    """Mean per-pixel CIELAB (D65) distance (analysis.py:162-174)."""
    xa, xb = _pair(a, b)
    return float(((_lab(xa) - _lab(xb)) ** 2).sum(dim=0).sqrt().mean())


def heatmap_u16(counts) -> np.ndarray:
    """Rescale a count plane to the full 16-bit range (analysis.py:177-184)."""
    c = np.asarray(counts, dtype=np.float64)
    peak = c.max()
    if peak <= 0:
        return np.zeros(c.shape, dtype=np.uint16)
    return np.floor(c / peak * 65535.0 + 0.5).astype(np.uint16)
