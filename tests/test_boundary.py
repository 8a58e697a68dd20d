"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/svdlut_b200.h declares, and maps invalid arguments onto the
reference's exception classes before touching a GPU; the Python mirror types
validate like the reference (core_types.py:62-255, errors.py:4-31)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2508_16121_b200 import _lib, errors
from paper_2508_16121_b200.core_types import (GridSet, GridWeights, Image, Lut2DSet, LutWeights,
                                              SvdLut)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build_library()
    return _lib.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "svdlut_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svdlut_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 18
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTS)


def test_version_and_status_names(lib):
    assert lib.svdlut_version() >= 10000
    names = [lib.svdlut_status_name(i).decode() for i in range(9)]
    assert names[:6] == ["OK", "DimensionMismatch", "DegenerateImage", "BadGridCount",
                         "BadVertexCount", "NonFiniteValue"]


def layout_bytes(dt, ds):
    from _layout import Layout

    return Layout(dt, ds).bytes


def test_table_sizes(lib):
    # d_t=33, d_s=17: 9 chunk planes of 32 x 35 cells (row stride 35 = 3 mod 8)
    # x 16 B, then the merged grid block
    assert 35 % 8 == 3
    assert lib.svdlut_table_bytes(33, 17) == layout_bytes(33, 17)
    assert layout_bytes(33, 17) >= 9 * 32 * 35 * 16 + 3 * 16 * 16 * 16 + 17 * 17 * 12 + 3 * 17 * 17 * 4
    for dt, ds in ((2, 2), (7, 8), (17, 8), (65, 33)):
        assert lib.svdlut_table_bytes(dt, ds) == layout_bytes(dt, ds)
    assert lib.svdlut_table_bytes(1, 17) == 0
    assert lib.svdlut_fast_supported(33, 17) == 1
    assert lib.svdlut_fast_supported(17, 8) == 1
    assert lib.svdlut_fast_supported(64, 17) == 0  # falls back to the exact kernel
    assert lib.svdlut_workspace_bytes(2, 2160, 3840, 33, 17) > 2 * lib.svdlut_table_bytes(33, 17)


NULL = ctypes.c_void_p(0)
FAKE = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first


@pytest.mark.parametrize("k,w,h,dt,ds,exc", [
    (4, 8, 8, 9, 5, errors.BadGridCount),
    (6, 1, 8, 9, 5, errors.DegenerateImage),
    (6, 8, 1, 9, 5, errors.DegenerateImage),
    (6, 8, 8, 1, 5, errors.BadVertexCount),
    (6, 8, 8, 9, 1, errors.BadVertexCount),
])
def test_c_abi_validation_maps_to_reference_errors(lib, k, w, h, dt, ds, exc):
    with pytest.raises(exc):
        _lib.call("svdlut_fused_fwd_exact", FAKE, 1, h, w, 0, h, FAKE, FAKE, FAKE, dt, FAKE, FAKE,
                  FAKE, k, ds, FAKE, NULL)


def test_c_abi_strip_outside_image(lib):
    with pytest.raises(errors.DimensionMismatch):
        _lib.call("svdlut_fused_fwd_exact", FAKE, 1, 10, 8, 5, 12, FAKE, FAKE, FAKE, 9, FAKE, FAKE,
                  FAKE, 6, 5, FAKE, NULL)


def test_c_abi_null_and_unsupported(lib):
    with pytest.raises(errors.InvalidArgument):
        _lib.call("svdlut_fused_fwd_exact", NULL, 1, 8, 8, 0, 8, FAKE, FAKE, FAKE, 9, FAKE, FAKE,
                  FAKE, 6, 5, FAKE, NULL)
    with pytest.raises(errors.Unsupported):
        _lib.call("svdlut_fused_fwd_packed", FAKE, 1, 8, 8, 0, 8, FAKE, 80, 17, FAKE, FAKE, 1 << 20,
                  NULL)
    with pytest.raises(errors.DimensionMismatch):
        _lib.call("svdlut_reconstruct", FAKE, FAKE, FAKE, 1, 9, 10, FAKE, NULL)  # rank > d
    _lib.call("svdlut_reconstruct", NULL, NULL, NULL, 0, 9, 3, NULL, NULL)  # empty batch: no-op


def test_mirror_types_validate_like_reference():
    img = Image(4, 3, np.zeros(36, np.float32))
    assert img.data.shape == (3, 3, 4) and not img.data.flags.writeable
    with pytest.raises(errors.DimensionMismatch):
        Image(4, 3, np.zeros(35, np.float32))
    with pytest.raises(errors.NonFiniteValue):
        Image(2, 2, np.full((3, 2, 2), np.nan, np.float32))
    with pytest.raises(errors.BadVertexCount):
        Lut2DSet(np.zeros((3, 3, 1, 1), np.float32))
    with pytest.raises(errors.DimensionMismatch):
        Lut2DSet(np.zeros((3, 2, 4, 4), np.float32))
    with pytest.raises(errors.DimensionMismatch):
        LutWeights(np.zeros((3, 2)), np.zeros(3))
    g = GridSet(np.zeros((6, 3, 5, 5)))
    assert (g.k, g.d_s) == (6, 5)
    assert GridWeights(np.zeros((6, 3)), np.zeros(6)).k == 6
    f = SvdLut(np.zeros((3, 3, 9, 2)), np.zeros((3, 3, 2)), np.zeros((3, 3, 2, 9)))
    assert (f.d_t, f.n_s) == (9, 2)
    with pytest.raises(errors.DimensionMismatch):
        SvdLut(np.zeros((3, 3, 9, 10)), np.zeros((3, 3, 10)), np.zeros((3, 3, 10, 9)))


def test_drop_in_validates_before_any_device_work():
    from paper_2508_16121_b200 import transform

    img = Image(6, 6, np.zeros((3, 6, 6), np.float32))
    luts = Lut2DSet(np.zeros((3, 3, 5, 5)))
    lw = LutWeights(np.eye(3), np.zeros(3))
    with pytest.raises(errors.BadGridCount):
        transform.fused_enhance(img, luts, lw, GridSet(np.zeros((4, 3, 5, 5))),
                                GridWeights(np.zeros((4, 3)), np.zeros(4)))
    with pytest.raises(errors.DimensionMismatch):
        transform.fused_enhance(img, luts, lw, GridSet(np.zeros((6, 3, 5, 5))),
                                GridWeights(np.zeros((3, 3)), np.zeros(3)))
    with pytest.raises(errors.DegenerateImage):
        transform.fused_enhance(Image(1, 6, np.zeros((3, 6, 1))), luts, lw,
                                GridSet(np.zeros((3, 3, 5, 5))),
                                GridWeights(np.zeros((3, 3)), np.zeros(3)))


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2508_16121_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "svdlut_oracle" not in src, f


def test_c_abi_widened_entries_validate_before_device_work(lib):
    """The sample-format, multi-stage, 3D-LUT and histogram entry points map
    bad arguments to the reference's error classes without touching a GPU."""
    with pytest.raises(errors.InvalidArgument):  # unknown sample format
        _lib.call("svdlut_fused_fwd_io", FAKE, 7, 1, 8, 8, 0, 8, FAKE, 33, 17, FAKE, 0, NULL, NULL)
    with pytest.raises(errors.InvalidArgument):  # L2-gradient format is an internal output only
        _lib.call("svdlut_fused_fwd_io", FAKE, 0, 1, 8, 8, 0, 8, FAKE, 33, 17, FAKE, 3, NULL, NULL)
    with pytest.raises(errors.DegenerateImage):
        _lib.call("svdlut_fused_fwd_io", FAKE, 1, 1, 1, 8, 0, 1, FAKE, 33, 17, FAKE, 1, NULL, NULL)
    with pytest.raises(errors.BadVertexCount):
        _lib.call("svdlut_slice_grids", FAKE, 1, 8, 8, 0, 8, FAKE, FAKE, FAKE, 6, 1, FAKE, NULL)
    with pytest.raises(errors.DimensionMismatch):
        _lib.call("svdlut_slice_grids", FAKE, 1, 8, 8, 0, 8, FAKE, FAKE, FAKE, 0, 5, FAKE, NULL)
    with pytest.raises(errors.BadVertexCount):
        _lib.call("svdlut_apply_lut3d", FAKE, 1, 8, 8, FAKE, 1, FAKE, NULL)
    with pytest.raises(errors.InvalidArgument):
        _lib.call("svdlut_apply_lut3d", NULL, 1, 8, 8, FAKE, 33, FAKE, NULL)
    with pytest.raises(errors.Unsupported):
        _lib.call("svdlut_occurrence", FAKE, 1, 8, 8, 2000, FAKE, NULL)
    with pytest.raises(errors.InvalidArgument):
        _lib.call("svdlut_occurrence", FAKE, 1, 8, 8, 33, NULL, NULL)
    # empty inputs are no-ops that never dereference the pointers
    _lib.call("svdlut_apply_lut3d", NULL, 0, 8, 8, NULL, 33, NULL, NULL)
    _lib.call("svdlut_fused_fwd_io", NULL, 1, 0, 8, 8, 0, 8, NULL, 33, 17, NULL, 1, NULL, NULL)
