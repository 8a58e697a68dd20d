"""ctypes binding of the C ABI in ``include/svdlut_b200.h``.

The shared library is built in-tree (``build.py``) for sm_100a.  There is no
fallback: if the library is missing or a CUDA device is absent, every entry
point raises — the product path never degrades to a CPU implementation.
"""

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVDLUT_LIB") or os.path.join(_HERE, "_lib", "libsvdlut_b200.so")

_lib = None

_vp = ctypes.c_void_p
_i = ctypes.c_int
_sz = ctypes.c_size_t

# name -> (restype, argtypes)
_SIGS = {
    "svdlut_version": (_i, []),
    "svdlut_last_error": (ctypes.c_char_p, []),
    "svdlut_status_name": (ctypes.c_char_p, [_i]),
    "svdlut_table_bytes": (_sz, [_i, _i]),
    "svdlut_fast_supported": (_i, [_i, _i]),
    "svdlut_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "svdlut_reconstruct": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp, _vp]),
    "svdlut_pack_tables": (_i, [_vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _i, _vp, _vp]),
    "svdlut_pack_tables_factors": (_i, [_vp, _vp, _vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _i,
                                        _vp, _vp]),
    "svdlut_fused_fwd_packed": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp, _sz, _vp]),
    "svdlut_fused_fwd_packed_ex": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp, _sz, _vp,
                                        _vp]),
    "svdlut_fused_fwd": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i,
                              _vp, _vp, _sz, _vp]),
    "svdlut_fused_fwd_exact": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i,
                                    _i, _vp, _vp]),
    "svdlut_indices": (_i, [_vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "svdlut_bwd_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i]),
    "svdlut_fused_bwd": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _i, _i, _vp,
                              _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "svdlut_reconstruct_bwd": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "svdlut_ctx_create": (_vp, [_i]),
    "svdlut_ctx_destroy": (None, [_vp]),
    "svdlut_enhance_host": (_i, [_vp, _vp, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _vp,
                                 _i, ctypes.POINTER(_i)]),
    "svdlut_reconstruct_host": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp]),
    "svdlut_slice_grids": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _i, _vp, _vp]),
    "svdlut_apply_lut2d": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp]),
    "svdlut_combine_slices": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "svdlut_apply_lut3d": (_i, [_vp, _i, _i, _i, _vp, _i, _vp, _vp]),
    "svdlut_fused_fwd_l2": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp, _vp,
                                 ctypes.c_float, _vp]),
    "svdlut_fused_bwd_packed": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp,
                                     _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "svdlut_fused_l2_step": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, ctypes.c_float, _vp, _vp, _i, _vp, _vp,
                                  _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "svdlut_occurrence": (_i, [_vp, _i, _i, _i, _i, _vp, _vp]),
    "svdlut_fused_fwd_io": (_i, [_vp, _i, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, _i, _vp, _vp]),
    "svdlut_enhance_host_io": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _i,
                                    _vp, _i, ctypes.POINTER(_i)]),
}

EXPORTS = tuple(_SIGS)

# svdlut_status -> exception class (errors.py of the reference, 1:1)
_STATUS = {
    1: errors.DimensionMismatch,
    2: errors.DegenerateImage,
    3: errors.BadGridCount,
    4: errors.BadVertexCount,
    5: errors.NonFiniteValue,
    6: errors.InvalidArgument,
    7: errors.Unsupported,
    8: errors.CudaError,
}


class NativeLibraryMissing(RuntimeError):
    """The sm_100a library has not been built (run __graft_entry__.build())."""


def load():
    """Load (once) and return the ctypes library; raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found; build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("SVDLUT_LIB") and not hasattr(L, name):
                continue  # development override: an older experimental build
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status):
    """Raise the exception class mapped to a non-zero svdlut_status."""
    if status == 0:
        return
    msg = load().svdlut_last_error().decode(errors="replace") or f"status {status}"
    raise _STATUS.get(status, errors.SvdLutError)(msg)


def call(name, *args):
    check(getattr(load(), name)(*args))
