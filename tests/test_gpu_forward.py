"""GPU parity of the forward path (fast fp32 kernel, f64 exact kernel, cell
selection, reconstruction) against the reference's golden vectors and the
pinned CPU oracle.  Tolerances (BASELINE.json north_star): indices bit-exact,
fp32 outputs within 1e-5 max-abs; the exact kernel is bitwise equal."""

import hashlib
import os

import numpy as np
import pytest

from conftest import golden_case, make_inputs

pytestmark = pytest.mark.gpu

TOL = 1e-5
NCPU = os.cpu_count() or 1


@pytest.fixture(scope="module")
def dev():
    import torch

    import __graft_entry__

    __graft_entry__.build_library()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda", 0)


def T(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def fast(c, dev, y0=0, h_total=None, rgb=None):
    from paper_2508_16121_b200 import device

    tables = device.pack_tables(T(c["lp"], dev), T(c["lw"], dev), T(c["lb"], dev), T(c["gp"], dev),
                                T(c["gw"], dev), T(c["gb"], dev))
    x = T(c["rgb"] if rgb is None else rgb, dev)
    return device.apply(x, tables, y0=y0, h_total=h_total)[0].cpu().numpy()


def exact(c, dev):
    from paper_2508_16121_b200 import device

    return device.apply_exact(T(c["rgb"], dev), T(c["lp"], dev), T(c["lw"], dev), T(c["lb"], dev),
                              T(c["gp"], dev), T(c["gw"], dev), T(c["gb"], dev))[0].cpu().numpy()


def oracle_out(oracle_mod, c, **kw):
    return oracle_mod.fused_fwd(c["rgb"], c["lp"], c["lw"], c["lb"], c["gp"], c["gw"], c["gb"],
                                threads=NCPU, **kw)


def test_exact_kernel_bit_identical_to_reference_golden(golden, dev):
    for name in golden["tr_cases"]:
        c = golden_case(golden, str(name))
        assert np.array_equal(exact(c, dev), c["want"]), name


def test_fast_kernel_within_tolerance_on_golden(golden, dev):
    from paper_2508_16121_b200 import device

    for name in golden["tr_cases"]:
        c = golden_case(golden, str(name))
        if not device.fast_supported(c["lp"].shape[2], c["gp"].shape[2]):
            continue
        err = np.abs(fast(c, dev) - c["want"]).max()
        assert err <= TOL, (name, err)


@pytest.mark.parametrize("d_t,d_s", [(2, 2), (3, 3), (7, 8), (9, 5), (16, 7), (17, 17), (33, 17),
                                     (64, 33), (65, 9)])
def test_cell_selection_bit_exact(dev, oracle_mod, d_t, d_s):
    from paper_2508_16121_b200 import device

    rng = np.random.default_rng(d_t * 100 + d_s)
    h, w = 37, 53
    rgb = rng.uniform(-0.2, 1.2, (3, h, w)).astype(np.float32)
    # sprinkle exact vertex hits k/(d-1), 0, 1 and 1-ulp
    hits = np.concatenate([np.arange(d_t) / np.float32(d_t - 1), np.arange(d_s) / np.float32(d_s - 1),
                           [0.0, 1.0, np.nextafter(np.float32(1), np.float32(0))]]).astype(np.float32)
    flat = rgb.reshape(-1)
    sel = rng.choice(flat.size, size=flat.size // 3, replace=False)
    flat[sel] = rng.choice(hits, size=sel.size)
    got = device.indices(T(rgb, dev), d_t, d_s)[0].cpu().numpy()
    want = oracle_mod.indices(rgb, d_t, d_s)
    assert np.array_equal(got, want)
    # strip of a taller image uses the global row normalisation
    got = device.indices(T(rgb[:, 10:20], dev), d_t, d_s, y0=10, h_total=h)[0].cpu().numpy()
    assert np.array_equal(got, want[:, 10:20])


def test_config2_4k_fast_and_exact_vs_oracle(dev, oracle_mod):
    """Config 2 (3x2160x3840 smooth field, defaults) at full size."""
    import torch

    from paper_2508_16121_b200 import device, synth

    case = synth.make_case(0)
    planes_d = device.reconstruct(T(case.u, dev), T(case.s, dev), T(case.vt, dev))
    planes = oracle_mod.reconstruct(case.u, case.s, case.vt)
    got_planes = planes_d[0].cpu().numpy()
    assert np.all(np.abs(got_planes - planes) <= np.spacing(np.abs(planes)))
    c = dict(rgb=case.rgb, lp=planes, lw=case.lw, lb=case.lb, gp=case.grid_planes, gw=case.gw,
             gb=case.gb)
    want = oracle_out(oracle_mod, c)
    got = fast(c, dev)
    err = float(np.abs(got - want).max())
    assert err <= TOL, err
    assert np.array_equal(exact(c, dev), want)
    # full-size index check
    idx = device.indices(T(case.rgb, dev), 33, 17)[0]
    want_idx = torch.from_numpy(oracle_mod.indices(case.rgb, 33, 17)).to(dev)
    assert torch.equal(idx, want_idx)


def test_uniform_noise_1080p_vs_oracle(dev, oracle_mod):
    """Worst-case locality (reference bench.synth_image-style noise)."""
    from paper_2508_16121_b200 import synth

    case = synth.uniform_case(3, 1080, 1920, low=-0.1, high=1.1)
    planes = oracle_mod.reconstruct(case.u, case.s, case.vt)
    c = dict(rgb=case.rgb, lp=planes, lw=case.lw, lb=case.lb, gp=case.grid_planes, gw=case.gw,
             gb=case.gb)
    want = oracle_out(oracle_mod, c)
    assert np.abs(fast(c, dev) - want).max() <= TOL


def test_row_strips_bitwise_equal_unsplit(dev):
    """Config-4 contract: strips (y0, h_total) reproduce the unsplit run bit for bit."""
    c = make_inputs(1000, 517, d_t=33, d_s=17, seed=9)
    full = fast(c, dev)
    bounds = [0, 64, 65, 200, 333, 517]
    parts = [fast(c, dev, y0=a, h_total=517, rgb=c["rgb"][:, a:b]) for a, b in zip(bounds, bounds[1:])]
    assert np.array_equal(np.concatenate(parts, axis=1), full)


def test_batch_equals_per_image(dev, oracle_mod):
    import torch

    from paper_2508_16121_b200 import device

    cs = [make_inputs(203, 77, d_t=17, d_s=8, k=9, seed=s) for s in range(3)]
    st = {k: T(np.stack([c[k] for c in cs]), dev) for k in cs[0]}
    out = device.fused_forward(st["rgb"], st["lp"], st["lw"], st["lb"], st["gp"], st["gw"], st["gb"])
    for i, c in enumerate(cs):
        assert torch.equal(out[i], T(fast(c, dev), dev))
        assert np.abs(out[i].cpu().numpy() - oracle_out(oracle_mod, c)).max() <= TOL


@pytest.mark.parametrize("w,h", [(2, 2), (3, 5), (129, 3), (1001, 17), (3839, 9)])
def test_odd_sizes(dev, oracle_mod, w, h):
    c = make_inputs(w, h, d_t=33, d_s=17, seed=w, low=-0.5, high=1.5)
    want = oracle_out(oracle_mod, c)
    assert np.abs(fast(c, dev) - want).max() <= TOL


def test_misaligned_buffers_use_scalar_path(dev, oracle_mod):
    import torch

    from paper_2508_16121_b200 import device

    c = make_inputs(64, 16, d_t=9, d_s=5, seed=4)
    buf = torch.empty(3 * 16 * 64 + 1, device=dev)
    x = buf[1:].view(1, 3, 16, 64)  # 4-byte offset: not 16 B aligned
    x.copy_(T(c["rgb"], dev)[None])
    tables = device.pack_tables(T(c["lp"], dev), T(c["lw"], dev), T(c["lb"], dev), T(c["gp"], dev),
                                T(c["gw"], dev), T(c["gb"], dev))
    got = device.apply(x, tables)[0].cpu().numpy()
    assert np.abs(got - oracle_out(oracle_mod, c)).max() <= TOL


def test_nonfinite_flag(dev):
    import torch

    from paper_2508_16121_b200 import device

    c = make_inputs(40, 8, d_t=9, d_s=5, seed=1)
    c["gw"] = np.full_like(c["gw"], 3e38)
    c["gp"] = np.abs(c["gp"]) + 1.0
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    tables = device.pack_tables(T(c["lp"], dev), T(c["lw"], dev), T(c["lb"], dev), T(c["gp"], dev),
                                T(c["gw"], dev), T(c["gb"], dev))
    device.apply(T(c["rgb"], dev), tables, nonfinite=flag)
    assert int(flag.item()) == 1
    c2 = make_inputs(40, 8, d_t=9, d_s=5, seed=1)
    flag.zero_()
    tables = device.pack_tables(*(T(c2[k], dev) for k in ("lp", "lw", "lb", "gp", "gw", "gb")))
    device.apply(T(c2["rgb"], dev), tables, nonfinite=flag)
    assert int(flag.item()) == 0


def test_reconstruct_golden(golden, dev):
    from paper_2508_16121_b200 import device

    for i in golden["rc_cases"]:
        got = device.reconstruct(T(golden[f"rc_{i}_u"], dev), T(golden[f"rc_{i}_s"], dev),
                                 T(golden[f"rc_{i}_vt"], dev))[0].cpu().numpy()
        want = golden[f"rc_{i}_planes"]
        assert np.all(np.abs(got - want) <= np.spacing(np.abs(want))), i


def test_config1_end_to_end_through_drop_in(golden, dev):
    """Reference run_model(720x480) output: exact drop-in reproduces its SHA-256."""
    from paper_2508_16121_b200 import svd, transform
    from paper_2508_16121_b200.core_types import (GridSet, GridWeights, Image, LutWeights,
                                                  SvdLut)

    rng = np.random.default_rng(0)
    img = Image(720, 480, rng.random((3, 480, 720), dtype=np.float32))
    luts = svd.reconstruct_lut(SvdLut(golden["c1_u"], golden["c1_s"], golden["c1_vt"]))
    assert np.array_equal(luts.planes, golden["c1_planes"])
    lw = LutWeights(golden["c1_lw"], golden["c1_lb"])
    grids, gw = GridSet(golden["c1_gp"]), GridWeights(golden["c1_gw"], golden["c1_gb"])
    y = transform.fused_enhance(img, luts, lw, grids, gw, exact=True)
    assert hashlib.sha256(np.ascontiguousarray(y.data).tobytes()).hexdigest() == str(golden["c1_out_sha"])
    allocs = []
    transform._raster_hook = allocs.append
    try:
        yf = transform.fused_enhance(img, luts, lw, grids, gw, threads=8)
    finally:
        transform._raster_hook = None
    assert allocs == [(3, 480, 720)]
    assert isinstance(yf, Image) and not yf.data.flags.writeable
    assert np.abs(yf.data[:, ::7, ::11] - golden["c1_out_sub"]).max() <= TOL
    assert np.abs(yf.data - y.data).max() <= TOL


def test_drop_in_nonfinite_raises(dev):
    from paper_2508_16121_b200 import errors, transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights

    c = make_inputs(16, 8, d_t=9, d_s=5, seed=2)
    with pytest.raises(errors.NonFiniteValue):
        transform.fused_enhance(Image(16, 8, c["rgb"]), Lut2DSet(c["lp"]),
                                LutWeights(np.full((3, 3), 3e38, np.float32), c["lb"]),
                                GridSet(np.abs(c["gp"]) + 1), GridWeights(np.full((6, 3), 3e38), c["gb"]))


def test_pack_from_factors_equals_reconstruct_then_pack(dev):
    import torch

    from paper_2508_16121_b200 import device, synth

    case = synth.make_batch([11, 12], h=64, w=96)
    t = {k: T(getattr(case, k), dev) for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    planes = device.reconstruct(t["u"], t["s"], t["vt"])
    a = device.pack_tables(planes, t["lw"], t["lb"], t["grid_planes"], t["gw"], t["gb"])
    b = device.pack_tables_factors(t["u"], t["s"], t["vt"], t["lw"], t["lb"], t["grid_planes"],
                                   t["gw"], t["gb"])
    assert torch.equal(a.buf, b.buf)


def test_column_table_and_inline_brackets_agree(dev, oracle_mod):
    """Very wide rows fall back to in-kernel column brackets (no smem table)."""
    c = make_inputs(20000, 3, d_t=17, d_s=8, seed=21)
    want = oracle_out(oracle_mod, c)
    assert np.abs(fast(c, dev) - want).max() <= TOL


@pytest.mark.parametrize("w,h", [(64, 2), (333, 100), (1000, 149), (517, 1203), (3840, 2160)])
def test_host_pipeline_equals_device_path(dev, w, h):
    """svdlut_enhance_host (H2D strips -> per-strip kernels -> D2H strips on
    three streams) returns what the device-resident kernel computes, for one
    and many strips, fewer rows than SMs, and rows that are not multiples of
    a chunk."""
    from paper_2508_16121_b200 import synth, transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights

    import oracle

    oracle.build()
    c = synth.make_case(7, h=h, w=w)
    planes = oracle.reconstruct(c.u, c.s, c.vt)
    args = (Lut2DSet(planes), LutWeights(c.lw, c.lb), GridSet(c.grid_planes), GridWeights(c.gw, c.gb))
    y = transform.fused_enhance(Image(w, h, c.rgb), *args)
    case = {"rgb": c.rgb, "lp": planes, "lw": c.lw, "lb": c.lb, "gp": c.grid_planes, "gw": c.gw, "gb": c.gb}
    want = fast(case, dev)
    assert np.abs(y.data - want).max() <= TOL
    assert np.mean(y.data != want) < 1e-4
    # repeated calls reuse the context's buffers
    y2 = transform.fused_enhance(Image(w, h, c.rgb), *args)
    assert np.array_equal(y.data, y2.data)
