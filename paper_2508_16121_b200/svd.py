"""Reference-facing ``reconstruct_lut`` (reference svd.py:210-220) on the GPU.

planes[c, p] = f32((f64 U * f64 S) @ f64 Vt) for the nine planes, computed by
the reconstruction kernel (svdlut_reconstruct).  Returns the Lut2DSet class of
the caller's package (ours or the reference's).
"""

import sys

import numpy as np

from .core_types import Lut2DSet as _Lut2DSet

__all__ = ["reconstruct_lut"]


def _lut_cls(svdlut):
    mod = sys.modules.get(type(svdlut).__module__)
    return getattr(mod, "Lut2DSet", _Lut2DSet)


def reconstruct_lut(svdlut):
    import torch

    from . import device

    dev = torch.device("cuda", torch.cuda.current_device())
    u = torch.from_numpy(np.ascontiguousarray(svdlut.u, np.float32)).to(dev)
    s = torch.from_numpy(np.ascontiguousarray(svdlut.s, np.float32)).to(dev)
    vt = torch.from_numpy(np.ascontiguousarray(svdlut.vt, np.float32)).to(dev)
    planes = device.reconstruct(u, s, vt)[0].cpu().numpy()
    return _lut_cls(svdlut)(planes)
