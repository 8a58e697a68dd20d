"""Multi-pass "original structure" (slice_grid2d, apply_lut2d, combine_slices,
naive_enhance) and the 3D-LUT baseline (apply_lut3d): the numpy oracle and the
GPU kernels (svdlut_naive.cu) against outputs of the reference itself
(tests/golden/make_naive_golden.py).  All bit-exact."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, make_inputs

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_naive_golden import LUT3D_CASES, NAIVE_CASES, lut3d_inputs  # noqa: E402


@pytest.fixture(scope="module")
def ngold():
    return np.load(os.path.join(ROOT, "tests", "golden", "naive_golden.npz"))


def _case(entry):
    name, w, h, dt, ds, k, seed, lo, hi = entry
    return name, make_inputs(w, h, d_t=dt, d_s=ds, k=k, seed=seed, low=lo, high=hi)


@pytest.mark.parametrize("entry", NAIVE_CASES, ids=[c[0] for c in NAIVE_CASES])
def test_oracle_naive_stages_match_reference(ngold, entry):
    from oracle import naive

    name, c = _case(entry)
    fs = naive.slice_grids(c["rgb"], c["gp"], c["gw"], c["gb"])
    base = naive.apply_lut2d(c["rgb"], c["lp"], c["lw"], c["lb"])
    assert np.array_equal(fs, ngold[f"{name}_fs"])
    assert np.array_equal(base, ngold[f"{name}_base"])
    assert np.array_equal(naive.combine_slices(base, fs), ngold[f"{name}_out"])


@pytest.mark.parametrize("entry", LUT3D_CASES, ids=[c[0] for c in LUT3D_CASES])
def test_oracle_lut3d_matches_reference(ngold, entry):
    from oracle import naive

    name, w, h, d, seed, lo, hi = entry
    rgb, cubes = lut3d_inputs(w, h, d, seed, lo, hi)
    assert np.array_equal(naive.apply_lut3d(rgb, cubes), ngold[f"{name}_out"])


def test_naive_errors_before_compute():
    """The reference's validation order (transform.py:160-163, :185-188,
    :206-207) — raised on the host, no GPU needed."""
    from paper_2508_16121_b200 import transform
    from paper_2508_16121_b200.core_types import (GridSet, GridWeights, Image, Lut2DSet,
                                                  LutWeights, SpatialFeatureMap)
    from paper_2508_16121_b200.errors import BadGridCount, DegenerateImage, DimensionMismatch

    c = make_inputs(8, 6, k=6)
    img = Image(8, 6, c["rgb"])
    luts, lw = Lut2DSet(c["lp"]), LutWeights(c["lw"], c["lb"])
    with pytest.raises(BadGridCount):
        transform.naive_enhance(img, luts, lw, GridSet(c["gp"][:4]), GridWeights(c["gw"][:4], c["gb"][:4]))
    with pytest.raises(DegenerateImage):
        transform.slice_grid2d(Image(1, 6, c["rgb"][:, :, :1]), GridSet(c["gp"]),
                               GridWeights(c["gw"], c["gb"]))
    with pytest.raises(DimensionMismatch):
        transform.slice_grid2d(img, GridSet(c["gp"]), GridWeights(c["gw"][:3], c["gb"][:3]))
    with pytest.raises(BadGridCount):
        transform.combine_slices(img, SpatialFeatureMap(np.zeros((4, 6, 8), np.float32)))
    with pytest.raises(DimensionMismatch):
        transform.combine_slices(img, SpatialFeatureMap(np.zeros((6, 5, 8), np.float32)))


@pytest.mark.gpu
@pytest.mark.parametrize("entry", NAIVE_CASES, ids=[c[0] for c in NAIVE_CASES])
def test_gpu_naive_stages_bit_exact(ngold, entry):
    import __graft_entry__
    from paper_2508_16121_b200 import transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights

    __graft_entry__.build_library()
    name, c = _case(entry)
    h, w = c["rgb"].shape[1:]
    img = Image(w, h, c["rgb"])
    luts, lw = Lut2DSet(c["lp"]), LutWeights(c["lw"], c["lb"])
    grids, gw = GridSet(c["gp"]), GridWeights(c["gw"], c["gb"])
    fs = transform.slice_grid2d(img, grids, gw)
    base = transform.apply_lut2d(img, luts, lw)
    assert np.array_equal(fs.data, ngold[f"{name}_fs"])
    assert np.array_equal(base.data, ngold[f"{name}_base"])
    assert np.array_equal(transform.combine_slices(base, fs).data, ngold[f"{name}_out"])
    assert np.array_equal(transform.naive_enhance(img, luts, lw, grids, gw).data, ngold[f"{name}_out"])


@pytest.mark.gpu
@pytest.mark.parametrize("entry", LUT3D_CASES, ids=[c[0] for c in LUT3D_CASES])
def test_gpu_lut3d_bit_exact(ngold, entry):
    import __graft_entry__
    from paper_2508_16121_b200 import transform
    from paper_2508_16121_b200.core_types import Image, Lut3D

    __graft_entry__.build_library()
    name, w, h, d, seed, lo, hi = entry
    rgb, cubes = lut3d_inputs(w, h, d, seed, lo, hi)
    y = transform.apply_lut3d(Image(w, h, rgb), Lut3D(cubes))
    assert np.array_equal(y.data, ngold[f"{name}_out"])


@pytest.mark.gpu
def test_gpu_naive_strip_and_batch_match_oracle():
    """Row strips (y0, h_total) and batches through the device API."""
    import torch

    import __graft_entry__
    from oracle import naive
    from paper_2508_16121_b200 import device

    __graft_entry__.build_library()
    c = make_inputs(50, 40, d_t=17, d_s=9, k=6, seed=9)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    fs_full = naive.slice_grids(c["rgb"], c["gp"], c["gw"], c["gb"])
    fs_strip = device.slice_grids(T(c["rgb"][:, 15:33])[None], T(c["gp"])[None], T(c["gw"])[None],
                                  T(c["gb"])[None], y0=15, h_total=40)
    assert np.array_equal(fs_strip[0].cpu().numpy(), fs_full[:, 15:33])
    x2 = T(np.stack([c["rgb"], c["rgb"][:, ::-1].copy()]))
    y = device.apply_lut2d(x2, T(np.stack([c["lp"]] * 2)), T(np.stack([c["lw"]] * 2)),
                           T(np.stack([c["lb"]] * 2)))
    assert np.array_equal(y[1].cpu().numpy(),
                          naive.apply_lut2d(c["rgb"][:, ::-1].copy(), c["lp"], c["lw"], c["lb"]))


from make_naive_golden import ANALYSIS_CASES, analysis_image  # noqa: E402


@pytest.mark.parametrize("entry", ANALYSIS_CASES, ids=[c[0] for c in ANALYSIS_CASES])
def test_oracle_occurrence_matches_reference(ngold, entry):
    from oracle import naive

    name, w, h, seed, d, lo, hi, smooth = entry
    cube = naive.occurrence(analysis_image(w, h, seed, lo, hi, smooth), d)
    assert np.array_equal(cube, ngold[f"{name}_cube"])


@pytest.mark.gpu
@pytest.mark.parametrize("entry", ANALYSIS_CASES, ids=[c[0] for c in ANALYSIS_CASES])
def test_gpu_occurrence_and_utilization_exact(ngold, entry):
    import __graft_entry__
    from paper_2508_16121_b200 import analysis
    from paper_2508_16121_b200.core_types import Image

    __graft_entry__.build_library()
    name, w, h, seed, d, lo, hi, smooth = entry
    img = Image(w, h, analysis_image(w, h, seed, lo, hi, smooth))
    occ = analysis.occurrence_stats([img, img], d)
    assert np.array_equal(occ.cube, 2 * ngold[f"{name}_cube"])
    assert occ.total == 2 * 8 * w * h
    util = [analysis.utilization_rate(img, d, m) for m in ("1d", "2d", "3d")]
    assert util == list(ngold[f"{name}_util"])


@pytest.mark.gpu
def test_gpu_image_metrics(ngold):
    import __graft_entry__
    from paper_2508_16121_b200 import analysis
    from paper_2508_16121_b200.core_types import Image

    __graft_entry__.build_library()
    a = Image(40, 30, analysis_image(40, 30, 11, 0.0, 1.0, False))
    b = Image(40, 30, analysis_image(40, 30, 12, -0.1, 1.1, False))
    assert abs(analysis.psnr(a, b) - float(ngold["an_psnr"])) <= 1e-9 * abs(float(ngold["an_psnr"]))
    assert abs(analysis.delta_e_ab(a, b) - float(ngold["an_delta_e"])) <= 1e-9 * float(ngold["an_delta_e"])
    assert analysis.psnr(a, a) == float("inf")


@pytest.mark.gpu
def test_gpu_naive_raster_hook_pattern():
    """naive_enhance allocates (K,H,W) then two (3,H,W) rasters through the
    raster hook, like the reference (tests/test_transform.py:321-329 there)."""
    import __graft_entry__
    from paper_2508_16121_b200 import transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights

    __graft_entry__.build_library()
    c = make_inputs(20, 12, k=6, seed=2)
    seen = []
    transform._raster_hook = seen.append
    try:
        transform.naive_enhance(Image(20, 12, c["rgb"]), Lut2DSet(c["lp"]), LutWeights(c["lw"], c["lb"]),
                                GridSet(c["gp"]), GridWeights(c["gw"], c["gb"]))
    finally:
        transform._raster_hook = None
    assert seen == [(6, 12, 20), (3, 12, 20), (3, 12, 20)]


@pytest.mark.gpu
@pytest.mark.parametrize("trial", range(10))
def test_gpu_fused_vs_naive_random_models(trial):
    """The reference's fused-vs-naive trials (d_t in [2,16], d_s in [2,8],
    K in {3,6,9}; tests/test_transform.py:281-296 there): the fast fused
    kernel within 1e-5 of the bit-exact naive stages, exact kernel within 1e-6."""
    import torch

    import __graft_entry__
    from paper_2508_16121_b200 import device

    __graft_entry__.build_library()
    rng = np.random.default_rng(100 + trial)
    d_t, d_s, k = int(rng.integers(2, 17)), int(rng.integers(2, 9)), int(rng.choice([3, 6, 9]))
    w, h = int(rng.integers(2, 70)), int(rng.integers(2, 50))
    c = make_inputs(w, h, d_t=d_t, d_s=d_s, k=k, seed=200 + trial)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()[None]  # noqa: E731
    x, lp, lw, lb, gp, gw, gb = (T(c[f]) for f in ("rgb", "lp", "lw", "lb", "gp", "gw", "gb"))
    naive = device.combine_slices(device.apply_lut2d(x, lp, lw, lb), device.slice_grids(x, gp, gw, gb))
    fast = device.apply(x, device.pack_tables(lp, lw, lb, gp, gw, gb))
    exact = device.apply_exact(x, lp, lw, lb, gp, gw, gb)
    assert float((fast - naive).abs().max()) <= 1e-5
    assert float((exact - naive).abs().max()) <= 1e-6


@pytest.mark.gpu
def test_gpu_bias_only_and_determinism():
    """Zero planes and grids: the output is exactly lb[c] + sum gb[k % 3 == c]
    (reference tests/test_transform.py:195-214 style); two launches are
    bitwise identical (the thread-count determinism test's analog)."""
    import torch

    import __graft_entry__
    from paper_2508_16121_b200 import device

    __graft_entry__.build_library()
    c = make_inputs(33, 17, d_t=9, d_s=5, k=6, seed=4)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()[None]  # noqa: E731
    x = T(c["rgb"])
    lb = torch.tensor([[0.25, -0.5, 0.125]], device="cuda")
    gb = torch.tensor([[0.5, 0.25, -0.25, 0.125, 1.0, 0.0625]], device="cuda")
    tables = device.pack_tables(T(np.zeros_like(c["lp"])), T(c["lw"]), lb, T(np.zeros_like(c["gp"])),
                                T(c["gw"]), gb)
    y = device.apply(x, tables)[0]
    for ch in range(3):
        want = float(lb[0, ch]) + float(gb[0, ch]) + float(gb[0, ch + 3])
        assert bool((y[ch] == want).all())
    tables = device.pack_tables(T(c["lp"]), T(c["lw"]), T(c["lb"]), T(c["gp"]), T(c["gw"]), T(c["gb"]))
    assert torch.equal(device.apply(x, tables), device.apply(x, tables))
