"""The drop-in plugin wires the B200 path into the reference package itself.

Runs in the build container, where /root/reference is importable (skipped
elsewhere; the GPU box never reads the reference).  Checks the patched names,
exception translation onto the reference's own classes, the raster-hook
contract and uninstall.  GPU numerics are covered by test_gpu_*.py.
"""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


@pytest.fixture
def ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_b200_tests")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import svdlut
    import svdlut.network
    import svdlut.svd
    import svdlut.transform

    return svdlut


def test_install_patches_and_uninstall_restores(ref):
    from paper_2508_16121_b200 import plugin

    orig = (ref.transform.fused_enhance, ref.network.fused_enhance, ref.svd.reconstruct_lut)
    h = plugin.install()
    try:
        assert ref.transform.fused_enhance is not orig[0]
        assert ref.network.fused_enhance is ref.transform.fused_enhance
        assert ref.svd.reconstruct_lut is not orig[2]
    finally:
        h.uninstall()
    assert (ref.transform.fused_enhance, ref.network.fused_enhance, ref.svd.reconstruct_lut) == orig


def test_errors_are_the_reference_classes(ref):
    from svdlut.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights
    from svdlut.errors import BadGridCount, DegenerateImage, DimensionMismatch

    from paper_2508_16121_b200 import plugin

    img = Image(6, 6, np.zeros((3, 6, 6), np.float32))
    luts = Lut2DSet(np.zeros((3, 3, 5, 5), np.float32))
    lw = LutWeights(np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    h = plugin.install()
    try:
        with pytest.raises(BadGridCount):
            ref.transform.fused_enhance(img, luts, lw, GridSet(np.zeros((4, 3, 5, 5), np.float32)),
                                        GridWeights(np.zeros((4, 3), np.float32), np.zeros(4, np.float32)))
        with pytest.raises(DimensionMismatch):
            ref.transform.fused_enhance(img, luts, lw, GridSet(np.zeros((6, 3, 5, 5), np.float32)),
                                        GridWeights(np.zeros((3, 3), np.float32), np.zeros(3, np.float32)))
        with pytest.raises(DegenerateImage):
            ref.transform.fused_enhance(Image(1, 4, np.zeros((3, 4, 1), np.float32)), luts, lw,
                                        GridSet(np.zeros((3, 3, 5, 5), np.float32)),
                                        GridWeights(np.zeros((3, 3), np.float32), np.zeros(3, np.float32)))
    finally:
        h.uninstall()


def test_raster_hook_sees_exactly_the_output(ref):
    import torch
    from svdlut.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights
    from svdlut.errors import SvdLutError

    from paper_2508_16121_b200 import plugin

    img = Image(32, 24, np.random.default_rng(0).random((3, 24, 32), dtype=np.float32))
    args = (img, Lut2DSet(np.zeros((3, 3, 9, 9), np.float32)),
            LutWeights(np.eye(3, dtype=np.float32), np.zeros(3, np.float32)),
            GridSet(np.zeros((6, 3, 5, 5), np.float32)),
            GridWeights(np.zeros((6, 3), np.float32), np.zeros(6, np.float32)))
    allocs = []
    h = plugin.install()
    ref.transform._raster_hook = allocs.append
    try:
        if torch.cuda.is_available():
            out = ref.transform.fused_enhance(*args)
            assert isinstance(out, Image)
        else:
            with pytest.raises(SvdLutError):  # no GPU here: fails loudly, no CPU fallback
                ref.transform.fused_enhance(*args)
    finally:
        ref.transform._raster_hook = None
        h.uninstall()
    assert allocs == [(3, 24, 32)]


def test_generator_option_patches_run_model(ref):
    from paper_2508_16121_b200 import plugin

    orig = ref.network.run_model
    h = plugin.install()
    assert ref.network.run_model is orig  # default: only the apply path
    h.uninstall()
    h = plugin.install(generator=True)
    try:
        assert ref.network.run_model is not orig
    finally:
        h.uninstall()
    assert ref.network.run_model is orig
