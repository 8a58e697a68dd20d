"""Reference-facing ``reconstruct_lut`` (reference svd.py:210-220) on the GPU.

planes[c, p] = f32((f64 U * f64 S) @ f64 Vt) for the nine planes, computed by
the reconstruction kernel (svdlut_reconstruct) behind the host-buffer entry
point svdlut_reconstruct_host.  Returns the Lut2DSet class of
the caller's package (ours or the reference's).
"""

import ctypes
import sys

import numpy as np

from .core_types import Lut2DSet as _Lut2DSet

__all__ = ["reconstruct_lut"]


def _lut_cls(svdlut):
    mod = sys.modules.get(type(svdlut).__module__)
    return getattr(mod, "Lut2DSet", _Lut2DSet)


def reconstruct_lut(svdlut):
    """planes = f32((f64 U * S) @ f64 Vt) per plane on the GPU (one H2D of the
    factors, svdlut_reconstruct, one D2H), through the C entry point
    svdlut_reconstruct_host."""
    from . import _lib, transform

    u = np.ascontiguousarray(svdlut.u, np.float32)
    s = np.ascontiguousarray(svdlut.s, np.float32)
    vt = np.ascontiguousarray(svdlut.vt, np.float32)
    d_t, n_s = u.shape[-2], u.shape[-1]
    planes = np.empty((3, 3, d_t, d_t), np.float32)
    ctx = transform._host_ctx(transform._current_device())
    ptr = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    _lib.call("svdlut_reconstruct_host", ctx, ptr(u), ptr(s), ptr(vt), 1, d_t, n_s, ptr(planes))
    return _lut_cls(svdlut)(planes)
