"""Exception classes of the apply path.

Names and hierarchy mirror the reference's ``svdlut.errors`` for the classes
this path can raise (reference errors.py:4-31), so callers written against the
reference catch the same names.  ``plugin.install`` re-raises them as the
reference's own classes when the drop-in is installed into ``svdlut``.
"""


class SvdLutError(Exception):
    """Base class of every error raised by this package."""


class DimensionMismatch(SvdLutError):
    """Declared dimensions disagree with the data they describe."""


class NonFiniteValue(SvdLutError):
    """A sample, table entry or weight is NaN or infinite."""


class BadVertexCount(SvdLutError):
    """A lookup table axis has fewer than two vertices."""


class DegenerateImage(SvdLutError):
    """Spatial coordinates are undefined for images narrower than 2 px."""


class BadGridCount(SvdLutError):
    """The grid count does not divide evenly into the three colour channels."""


class InvalidArgument(SvdLutError):
    """A device buffer is missing, misaligned or too small (C ABI misuse)."""


class Unsupported(SvdLutError):
    """The request exceeds what the selected kernel supports."""


class CudaError(SvdLutError):
    """The CUDA runtime reported an error."""
