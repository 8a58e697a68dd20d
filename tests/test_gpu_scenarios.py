"""Model-level scenarios of the reference's operator tests (reference
tests/test_transform.py:195-296: zero grids, zero model, identity-style
model, thread independence, fused vs multi-stage on random small models)
run through the drop-in operators on the GPU."""

import numpy as np
import pytest

from conftest import make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    import torch

    import __graft_entry__

    __graft_entry__.build_library()
    assert torch.cuda.is_available()
    from paper_2508_16121_b200 import core_types, transform

    return transform, core_types


def _model(c, ct):
    return (ct.Lut2DSet(c["lp"]), ct.LutWeights(c["lw"], c["lb"]), ct.GridSet(c["gp"]),
            ct.GridWeights(c["gw"], c["gb"]))


def _zero_grids(ct, k, d):
    return ct.GridSet(np.zeros((k, 3, d, d), np.float32)), ct.GridWeights(np.zeros((k, 3), np.float32),
                                                                          np.zeros(k, np.float32))


def _identity_luts(ct, d):
    """Channel c reproduced through one pair whose plane is a ramp along c's axis:
    r via pair rg (first axis), g via pair gb (first axis), b via pair rb (second axis)."""
    ramp = np.arange(d, dtype=np.float32) / np.float32(d - 1)
    planes = np.zeros((3, 3, d, d), np.float32)
    w = np.zeros((3, 3), np.float32)
    planes[0, 0] = ramp[:, None]
    w[0, 0] = 1
    planes[1, 2] = ramp[:, None]
    w[1, 2] = 1
    planes[2, 1] = ramp[None, :]
    w[2, 1] = 1
    return ct.Lut2DSet(planes), ct.LutWeights(w, np.zeros(3, np.float32))


def test_zero_grids_equal_lut_only(ops):
    transform, ct = ops
    c = make_inputs(16, 16, d_t=9, d_s=5, k=6, seed=32)
    img = ct.Image(16, 16, c["rgb"])
    luts, lw = ct.Lut2DSet(c["lp"]), ct.LutWeights(c["lw"], c["lb"])
    grids, gw = _zero_grids(ct, 6, 5)
    fused = transform.fused_enhance(img, luts, lw, grids, gw)
    lut_only = transform.apply_lut2d(img, luts, lw)
    assert np.abs(fused.data - lut_only.data).max() <= 1e-6


def test_zero_model_gives_zero_output(ops):
    transform, ct = ops
    c = make_inputs(6, 6, d_t=5, d_s=5, k=6, seed=46)
    img = ct.Image(6, 6, c["rgb"])
    luts = ct.Lut2DSet(np.zeros((3, 3, 5, 5), np.float32))
    lw = ct.LutWeights(np.zeros((3, 3), np.float32), np.zeros(3, np.float32))
    grids, gw = _zero_grids(ct, 6, 5)
    assert np.all(transform.fused_enhance(img, luts, lw, grids, gw).data == 0)
    assert np.all(transform.naive_enhance(img, luts, lw, grids, gw).data == 0)


@pytest.mark.parametrize("d", [2, 9, 33])
def test_identity_style_model_reproduces_input(ops, d):
    transform, ct = ops
    rng = np.random.default_rng(47)
    x = rng.random((3, 9, 13), dtype=np.float32)
    img = ct.Image(13, 9, x)
    luts, lw = _identity_luts(ct, d)
    grids, gw = _zero_grids(ct, 3, 5)
    assert np.abs(transform.fused_enhance(img, luts, lw, grids, gw).data - x).max() <= 1e-6
    assert np.abs(transform.naive_enhance(img, luts, lw, grids, gw).data - x).max() <= 1e-6


def test_thread_argument_does_not_change_bits(ops):
    transform, ct = ops
    c = make_inputs(64, 48, d_t=9, d_s=5, k=6, seed=48)
    img = ct.Image(64, 48, c["rgb"])
    serial = transform.fused_enhance(img, *_model(c, ct), threads=1)
    threaded = transform.fused_enhance(img, *_model(c, ct), threads=4)
    assert np.array_equal(serial.data, threaded.data)


def test_random_small_models_fused_vs_multistage(ops):
    """Random sizes 2..32 px, d_t 2..16, d_s 2..8, K in {3, 6, 9}."""
    transform, ct = ops
    rng = np.random.default_rng(53)
    worst = 0.0
    for trial in range(10):
        w, h = int(rng.integers(2, 33)), int(rng.integers(2, 33))
        d_t, d_s, k = int(rng.integers(2, 17)), int(rng.integers(2, 9)), 3 * int(rng.integers(1, 4))
        c = make_inputs(w, h, d_t=d_t, d_s=d_s, k=k, seed=100 + trial)
        img = ct.Image(w, h, c["rgb"])
        fused = transform.fused_enhance(img, *_model(c, ct))
        naive = transform.naive_enhance(img, *_model(c, ct))
        worst = max(worst, float(np.abs(fused.data - naive.data).max()))
    assert worst <= 1e-5


def test_graph_replay_after_wider_eager_launch(ops):
    """a CUDA graph captured at 720x480, then an eager 4K launch of
    the same kernel instantiation, then the graph replayed: the kernel's
    dynamic shared-memory limit is set once to the maximum, so the replay
    still launches and reproduces its first output bit for bit."""
    import torch

    from paper_2508_16121_b200 import device, network, synth

    gen = network.Generator(network.random_init(0), device="cuda")
    x = torch.from_numpy(np.random.default_rng(0).random((1, 3, 480, 720), dtype=np.float32)).cuda()
    run = gen.graphed(x.shape)
    first = run(x).clone()
    case = synth.make_case(1)
    t = {k: torch.from_numpy(np.ascontiguousarray(getattr(case, k))).cuda()
         for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    tables = device.pack_tables_factors(*(t[k] for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")))
    device.apply(torch.from_numpy(case.rgb).cuda()[None], tables)  # eager, 3840 wide
    torch.cuda.synchronize()
    again = run(x)
    torch.cuda.synchronize()
    assert torch.equal(first, again)
