"""Host-side value types of the apply path.

Same names, fields, shapes and invariants as the reference's
``svdlut.core_types`` (reference core_types.py:62-255) so code written against
the reference runs unchanged: float32, C-contiguous, read-only arrays, finite
values checked at construction (``NonFiniteValue``), shape errors as
``DimensionMismatch`` / ``BadVertexCount``.

One addition: ``Image._trusted`` builds an Image whose finiteness was already
established on the device (the fused kernel ORs a non-finite flag), so the
drop-in does not re-scan a 100 MB raster on the host.
"""

from dataclasses import dataclass

import numpy as np

from .errors import BadVertexCount, DimensionMismatch, NonFiniteValue

__all__ = ["Image", "Lut2DSet", "LutWeights", "GridSet", "GridWeights", "SvdLut", "Lut3D",
           "SpatialFeatureMap"]


def _ro_f32(a):
    """float32, C-contiguous, read-only view (copies only when needed)."""
    arr = np.ascontiguousarray(a, dtype=np.float32)
    arr.flags.writeable = False
    return arr


def _require_finite(arr, what):
    # min/max propagate NaN and expose +-inf without a full boolean temporary
    if arr.size and not (np.isfinite(arr.min()) and np.isfinite(arr.max())):
        raise NonFiniteValue(f"{what} contains a NaN or infinite entry")


def _store(obj, **fields):
    for k, v in fields.items():
        object.__setattr__(obj, k, v)


@dataclass(frozen=True)
class Image:
    """Planar RGB raster (3, height, width); flat input of 3*w*h is reshaped."""

    width: int
    height: int
    data: np.ndarray

    def __post_init__(self):
        self._shape_and_freeze()
        _require_finite(self.data, "image data")

    def _shape_and_freeze(self):
        if not (isinstance(self.width, int) and isinstance(self.height, int)):
            raise DimensionMismatch("width and height must be integers")
        if min(self.width, self.height) < 1:
            raise DimensionMismatch("width and height must be >= 1")
        d = np.asarray(self.data, dtype=np.float32)
        n = 3 * self.width * self.height
        if d.size != n:
            raise DimensionMismatch(
                f"data has {d.size} samples but a {self.width}x{self.height} image needs {n}")
        _store(self, data=_ro_f32(d.reshape(3, self.height, self.width)))

    @classmethod
    def _trusted(cls, width, height, data):
        """Construct without the host finiteness scan (device already checked)."""
        obj = object.__new__(cls)
        _store(obj, width=width, height=height, data=data)
        obj._shape_and_freeze()
        return obj

    @property
    def channels(self) -> int:
        return 3


@dataclass(frozen=True)
class Lut2DSet:
    """planes[c][p] (3, 3, d, d): output channel c, input pair p in (rg, rb, gb)."""

    planes: np.ndarray

    def __post_init__(self):
        p = np.asarray(self.planes, dtype=np.float32)
        if p.ndim != 4 or p.shape[:2] != (3, 3) or p.shape[2] != p.shape[3]:
            raise DimensionMismatch(f"expected (3, 3, d, d) planes, got {p.shape}")
        if p.shape[2] < 2:
            raise BadVertexCount("2D LUT needs at least 2 vertices per axis")
        _store(self, planes=_ro_f32(p))
        _require_finite(self.planes, "2D LUT planes")

    @property
    def d_t(self) -> int:
        return self.planes.shape[2]


@dataclass(frozen=True)
class LutWeights:
    """w (3, 3): per output channel the (rg, rb, gb) plane weights; b (3,) biases."""

    w: np.ndarray
    b: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.w, dtype=np.float32)
        b = np.asarray(self.b, dtype=np.float32)
        if w.shape != (3, 3) or b.shape != (3,):
            raise DimensionMismatch(f"expected w (3,3) and b (3,), got {w.shape} {b.shape}")
        _store(self, w=_ro_f32(w), b=_ro_f32(b))
        _require_finite(self.w, "LUT weights")
        _require_finite(self.b, "LUT biases")


@dataclass(frozen=True)
class GridSet:
    """planes (k, 3, d, d): per grid the (xy, xc, yc) planes; guide = channel k % 3."""

    planes: np.ndarray

    def __post_init__(self):
        p = np.asarray(self.planes, dtype=np.float32)
        if p.ndim != 4 or p.shape[1] != 3 or p.shape[2] != p.shape[3]:
            raise DimensionMismatch(f"expected (k, 3, d, d) planes, got {p.shape}")
        if p.shape[0] < 1:
            raise DimensionMismatch("need at least one grid")
        if p.shape[2] < 2:
            raise BadVertexCount("grid needs at least 2 vertices per axis")
        _store(self, planes=_ro_f32(p))
        _require_finite(self.planes, "grid planes")

    @property
    def k(self) -> int:
        return self.planes.shape[0]

    @property
    def d_s(self) -> int:
        return self.planes.shape[2]


@dataclass(frozen=True)
class GridWeights:
    """w (k, 3): per grid (xy, xc, yc) weights; b (k,) biases."""

    w: np.ndarray
    b: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.w, dtype=np.float32)
        b = np.asarray(self.b, dtype=np.float32)
        if w.ndim != 2 or w.shape[1] != 3 or b.shape != (w.shape[0],):
            raise DimensionMismatch(f"expected w (k,3) and b (k,), got {w.shape} {b.shape}")
        _store(self, w=_ro_f32(w), b=_ro_f32(b))
        _require_finite(self.w, "grid weights")
        _require_finite(self.b, "grid biases")

    @property
    def k(self) -> int:
        return self.w.shape[0]


@dataclass(frozen=True)
class SvdLut:
    """Per plane U (d, n), S (n,), Vt (n, d): u (3,3,d,n), s (3,3,n), vt (3,3,n,d)."""

    u: np.ndarray
    s: np.ndarray
    vt: np.ndarray

    def __post_init__(self):
        u, s, vt = (np.asarray(a, dtype=np.float32) for a in (self.u, self.s, self.vt))
        if u.ndim != 4 or u.shape[:2] != (3, 3):
            raise DimensionMismatch(f"expected u (3, 3, d, n), got {u.shape}")
        d, n = u.shape[2:]
        if s.shape != (3, 3, n) or vt.shape != (3, 3, n, d):
            raise DimensionMismatch(
                f"inconsistent factor shapes u={u.shape} s={s.shape} vt={vt.shape}")
        if d < 2:
            raise BadVertexCount("factored LUT needs at least 2 vertices per axis")
        if not 1 <= n <= d:
            raise DimensionMismatch(f"rank {n} outside 1..{d}")
        _store(self, u=_ro_f32(u), s=_ro_f32(s), vt=_ro_f32(vt))
        for arr, what in ((self.u, "U factors"), (self.s, "singular values"),
                          (self.vt, "Vt factors")):
            _require_finite(arr, what)

    @property
    def d_t(self) -> int:
        return self.u.shape[2]

    @property
    def n_s(self) -> int:
        return self.u.shape[3]


@dataclass(frozen=True)
class Lut3D:
    """tables[c][i_r][i_g][i_b] (3, d, d, d): one cube per output channel
    (reference core_types.py:96-116)."""

    tables: np.ndarray

    def __post_init__(self):
        t = np.asarray(self.tables, dtype=np.float32)
        if t.ndim != 4 or t.shape[0] != 3 or not (t.shape[1] == t.shape[2] == t.shape[3]):
            raise DimensionMismatch(f"expected (3, d, d, d) tables, got {t.shape}")
        if t.shape[1] < 2:
            raise BadVertexCount("3D LUT needs at least 2 vertices per axis")
        _store(self, tables=_ro_f32(t))
        _require_finite(self.tables, "3D LUT tables")

    @property
    def d_t(self) -> int:
        return self.tables.shape[1]


@dataclass(frozen=True)
class SpatialFeatureMap:
    """k per-grid slicing maps over the image plane, (k, h, w)
    (reference transform.py:60-76)."""

    data: np.ndarray

    def __post_init__(self):
        d = np.asarray(self.data, dtype=np.float32)
        if d.ndim != 3:
            raise DimensionMismatch(f"expected (k, h, w), got {d.shape}")
        _store(self, data=_ro_f32(d))

    @property
    def k(self) -> int:
        return self.data.shape[0]
