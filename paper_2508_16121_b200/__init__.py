"""B200-native (sm_100a) SVDLUT apply path: fused bilateral-grid slicing +
2D-LUT transform, LUT reconstruction from SVD factors, and their backward.

Reference-facing drop-ins (same signatures as the reference ``svdlut``):
    transform.fused_enhance, svd.reconstruct_lut
Device-tensor API (inputs resident in HBM): ``device``
Training: ``autograd.SvdLutApply``; multi-GPU sharding: ``parallel``.
"""

from . import errors
from .core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights, SvdLut
from .errors import SvdLutError

__version__ = "0.1.0"

__all__ = [
    "errors", "GridSet", "GridWeights", "Image", "Lut2DSet", "LutWeights", "SvdLut",
    "SvdLutError", "native_library",
]


def native_library():
    """Load the sm_100a C-ABI library (raises if it was not built)."""
    from . import _lib

    return _lib.load()
