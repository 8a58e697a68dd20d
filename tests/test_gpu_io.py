"""PNM sample formats fused into the forward kernel (svdlut_io.cuh):
decode of pnm.load (reference pnm.py:72-80) and quantization of pnm.save
(pnm.py:83-108) must be bit-exact; the fused u8/u16 path must equal the f32
path followed by that quantization, bit for bit.

The decode/quantize stages are isolated with an *exact identity* table set:
all LUT weights and biases zero, grid k (k < 3) = the identity ramp j/16 on
its xc plane with weights (0, 1, 0).  With d_s - 1 = 16 (a power of two) the
fast kernel computes y = (jc + ec) / 16 = x exactly.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch

    import __graft_entry__

    __graft_entry__.build_library()
    assert torch.cuda.is_available()
    return torch.device("cuda", 0)


def identity_tables(dev, d_t=33, d_s=17):
    import torch

    from paper_2508_16121_b200 import device

    lp = torch.zeros((1, 3, 3, d_t, d_t), device=dev)
    lw = torch.zeros((1, 3, 3), device=dev)
    lb = torch.zeros((1, 3), device=dev)
    gp = torch.zeros((1, 3, 3, d_s, d_s), device=dev)
    ramp = torch.arange(d_s, dtype=torch.float32, device=dev) / (d_s - 1)
    for k in range(3):
        gp[0, k, 1, :, :] = ramp[None, :]
    gw = torch.zeros((1, 3, 3), device=dev)
    gw[0, :, 1] = 1.0
    gb = torch.zeros((1, 3), device=dev)
    return device.pack_tables(lp, lw, lb, gp, gw, gb)


def real_tables(dev, seed=0):
    import torch

    from paper_2508_16121_b200 import device, synth

    c = synth.make_case(seed, h=8, w=8)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)[None]  # noqa: E731
    planes = device.reconstruct(T(c.u), T(c.s), T(c.vt))
    return device.pack_tables(planes, T(c.lw), T(c.lb), T(c.grid_planes), T(c.gw), T(c.gb))


def to_be_bytes(v):
    """uint16 (H, W, 3) -> (H, W, 6) uint8 big-endian bytes."""
    return np.ascontiguousarray(v.astype(">u2")).view(np.uint8).reshape(v.shape[0], v.shape[1], 6)


def from_be_bytes(b):
    return b.reshape(b.shape[0], b.shape[1], 3, 2).copy().view(">u2")[..., 0].astype(np.uint16)


def ref_quantize(x, maxval):
    """pnm._quantize (pnm.py:83-86)."""
    return np.floor(np.clip(x.astype(np.float64), 0.0, 1.0) * maxval + 0.5)


def test_identity_tables_are_exact(dev):
    import torch

    from paper_2508_16121_b200 import device

    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.random((1, 3, 37, 64), dtype=np.float32)).to(dev)
    y = device.apply(x, identity_tables(dev))
    assert torch.equal(x, y)


@pytest.mark.parametrize("fmt,maxval", [("u8", 255), ("u16be", 65535)])
def test_decode_every_sample_value_bit_exact(dev, fmt, maxval):
    import torch

    from paper_2508_16121_b200 import device

    n = maxval + 1
    w = 128 if n == 256 else 256  # at least 2 rows
    h = n // w
    v = np.arange(n, dtype=np.uint16).reshape(h, w)
    img = np.stack([v, v[::-1], np.roll(v, 7)], axis=-1)  # (h, w, 3)
    raw = img.astype(np.uint8) if fmt == "u8" else to_be_bytes(img)
    y = device.apply_io(torch.from_numpy(raw).to(dev), identity_tables(dev), in_fmt=fmt, out_fmt="f32")
    want = (img.astype(np.float64) / maxval).astype(np.float32).transpose(2, 0, 1)
    assert np.array_equal(y[0].cpu().numpy(), want)


@pytest.mark.parametrize("fmt,maxval", [("u8", 255), ("u16be", 65535)])
def test_quantize_bit_exact_at_boundaries(dev, fmt, maxval):
    """x at every (n + 1/2)/maxval boundary +- a few ulps, 0, 1, out of range."""
    import torch

    from paper_2508_16121_b200 import device

    n = np.arange(0, maxval, max(1, maxval // 4096), dtype=np.float64)
    mid = ((n + 0.5) / maxval).astype(np.float32)
    xs = [mid]
    up, down = mid, mid
    for _ in range(3):  # +-1..3 ulps around each boundary
        up = np.nextafter(up, np.float32(2))
        down = np.nextafter(down, np.float32(-1))
        xs += [up, down]
    rng = np.random.default_rng(3)
    xs.append(rng.random(20000, dtype=np.float32))
    xs.append(np.array([0.0, 1.0, -0.0, -1e-9, 1.0000001, -5.0, 7.0, 0.5, 1e-30], np.float32))
    flat = np.concatenate(xs).astype(np.float32)
    w = 128
    flat = np.concatenate([flat, np.zeros((-flat.size) % (3 * w), np.float32)])
    x = flat.reshape(3, -1, w)
    y = device.apply_io(torch.from_numpy(x[None]).to(dev), identity_tables(dev), in_fmt="f32",
                        out_fmt=fmt)
    got = y[0].cpu().numpy()
    got = got if fmt == "u8" else from_be_bytes(got)
    want = ref_quantize(x.transpose(1, 2, 0), maxval)
    assert np.array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("fmt", ["u8", "u16be"])
@pytest.mark.parametrize("w", [64, 61])
def test_fused_io_equals_f32_path_then_quantize(dev, fmt, w):
    """u8/u16 in and out == decode -> fast f32 kernel -> quantize, bitwise;
    w=61 exercises the unaligned scalar path."""
    import torch

    from paper_2508_16121_b200 import device

    maxval = 255 if fmt == "u8" else 65535
    tables = real_tables(dev)
    rng = np.random.default_rng(5)
    img = rng.integers(0, maxval + 1, (45, w, 3)).astype(np.uint16)
    raw = img.astype(np.uint8) if fmt == "u8" else to_be_bytes(img)
    xq = torch.from_numpy(raw).to(dev)
    got = device.apply_io(xq, tables, in_fmt=fmt, out_fmt=fmt)[0].cpu().numpy()
    got = got if fmt == "u8" else from_be_bytes(got)
    x = torch.from_numpy((img.astype(np.float64) / maxval).astype(np.float32).transpose(2, 0, 1).copy())
    y = device.apply(x[None].to(dev), tables)[0].cpu().numpy()
    assert np.array_equal(got.astype(np.float64), ref_quantize(y.transpose(1, 2, 0), maxval))
    yd = device.apply_io(xq, tables, in_fmt=fmt, out_fmt="f32")[0].cpu().numpy()
    assert np.array_equal(yd, y)


def test_enhance_payload_host_entry(dev):
    """transform.enhance_payload (host numpy payload in/out through
    svdlut_enhance_host_io) == the device path, and within +-1 of the oracle
    (f64 reference semantics) after quantization."""
    import torch

    import oracle
    from paper_2508_16121_b200 import device, synth, transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, LutWeights
    from paper_2508_16121_b200.core_types import Lut2DSet

    oracle.build()
    c = synth.make_case(2, h=120, w=200)
    planes = oracle.reconstruct(c.u, c.s, c.vt)
    payload = np.ascontiguousarray(np.clip(np.round(c.rgb.transpose(1, 2, 0) * 255), 0, 255).astype(np.uint8))
    got = transform.enhance_payload(payload, Lut2DSet(planes), LutWeights(c.lw, c.lb),
                                    GridSet(c.grid_planes), GridWeights(c.gw, c.gb))
    assert got.dtype == np.uint8 and got.shape == payload.shape
    x = (payload.astype(np.float64) / 255).astype(np.float32).transpose(2, 0, 1).copy()
    ref = oracle.fused_fwd(x, planes, c.lw, c.lb, c.grid_planes, c.gw, c.gb)
    diff = np.abs(got.astype(np.int64) - ref_quantize(ref.transpose(1, 2, 0), 255).astype(np.int64))
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)[None]  # noqa: E731
    tables = device.pack_tables(T(planes), T(c.lw), T(c.lb), T(c.grid_planes), T(c.gw), T(c.gb))
    dv = device.apply_io(torch.from_numpy(payload).to(dev), tables, in_fmt="u8", out_fmt="u8")
    assert np.array_equal(dv[0].cpu().numpy(), got)
    got16 = transform.enhance_payload(payload, Lut2DSet(planes), LutWeights(c.lw, c.lb),
                                      GridSet(c.grid_planes), GridWeights(c.gw, c.gb), out_bits=16)
    assert got16.dtype == np.dtype(">u2")
    d16 = np.abs(got16.astype(np.int64) - ref_quantize(ref.transpose(1, 2, 0), 65535).astype(np.int64))
    assert d16.max() <= 1


@pytest.mark.parametrize("fmt", ["u8", "u16be"])
@pytest.mark.parametrize("w,h", [(1001, 777), (3840, 2160)])
def test_enhance_payload_many_strips_equals_device(dev, fmt, w, h):
    """Large payloads travel as many strips through the streamed kernel; the
    result is the device path's bit for bit (w=1001: unaligned rows)."""
    import torch

    from paper_2508_16121_b200 import device, synth, transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, Lut2DSet, LutWeights

    c = synth.make_case(4, h=8, w=8)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)[None]  # noqa: E731
    planes = device.reconstruct(T(c.u), T(c.s), T(c.vt))
    tables = device.pack_tables(planes, T(c.lw), T(c.lb), T(c.grid_planes), T(c.gw), T(c.gb))
    maxval = 255 if fmt == "u8" else 65535
    rng = np.random.default_rng(9)
    img = rng.integers(0, maxval + 1, (h, w, 3)).astype(np.uint16)
    payload = img.astype(np.uint8) if fmt == "u8" else img.astype(">u2")
    got = transform.enhance_payload(payload, Lut2DSet(planes[0].cpu().numpy()), LutWeights(c.lw, c.lb),
                                    GridSet(c.grid_planes), GridWeights(c.gw, c.gb))
    raw = payload if fmt == "u8" else to_be_bytes(img)
    dv = device.apply_io(torch.from_numpy(np.ascontiguousarray(raw)).to(dev), tables, in_fmt=fmt,
                         out_fmt=fmt)[0].cpu().numpy()
    dv = dv if fmt == "u8" else from_be_bytes(dv)
    assert np.array_equal(np.asarray(got).astype(np.int64), dv.astype(np.int64))


@pytest.mark.parametrize("pinned_in,pinned_out", [(False, False), (True, False), (False, True)])
def test_enhance_payload_pageable_buffers(dev, pinned_in, pinned_out):
    """Pageable payloads (plain numpy arrays) travel through the context's
    page-locked strip slots; the result equals the page-locked path bit for bit."""
    import torch

    from paper_2508_16121_b200 import device, synth, transform
    from paper_2508_16121_b200.core_types import GridSet, GridWeights, Lut2DSet, LutWeights

    c = synth.make_case(6, h=8, w=8)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)[None]  # noqa: E731
    planes = device.reconstruct(T(c.u), T(c.s), T(c.vt))
    model = (Lut2DSet(planes[0].cpu().numpy()), LutWeights(c.lw, c.lb), GridSet(c.grid_planes),
             GridWeights(c.gw, c.gb))
    h, w = 1499, 2001
    rng = np.random.default_rng(13)
    img = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    src = img
    if pinned_in:
        src = torch.empty((h, w, 3), dtype=torch.uint8, pin_memory=True).numpy()
        src[...] = img
    out = (torch.empty((h, w, 3), dtype=torch.uint8, pin_memory=True).numpy() if pinned_out
           else np.empty((h, w, 3), np.uint8))
    got = transform.enhance_payload(src, *model, out=out)
    assert got is out
    ref_in = torch.empty((h, w, 3), dtype=torch.uint8, pin_memory=True).numpy()
    ref_in[...] = img
    want = transform.enhance_payload(ref_in, *model)
    assert np.array_equal(got, want)
