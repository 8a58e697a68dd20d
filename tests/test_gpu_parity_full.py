"""Full-size parity of the product kernels (VERDICT r1 "parity holes").

* Cell selection INSIDE the fused forward kernel: hand-built packed tables in
  which one coefficient of every cell is its own id and everything else is
  zero, so the kernel's output is the id of the cell it selected.  Channel 0
  carries pair rg's ids, channel 1 pair rb's, channel 2 pair gb's (one launch
  covers the shared-memory and the texture-path planes); a second table puts
  the ids into the merged xc grid cells, so the output reveals (x-cell, guide
  cell) per channel.  Compared with the index oracle (interp.py:35-45,
  transform.py:144-149) on the config-2 4K image with vertex hits, on an 8K
  row strip with y0 > 0 and on the 17/8 and generic specialisations.
* BASELINE configs 3, 4, 5 at their stated sizes vs the CPU oracle.
"""

import numpy as np
import pytest

from _layout import Layout, empty_table, write_cells

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def dev():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build_library()
    return torch.device("cuda", 0)


def T(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def with_vertex_hits(rgb, d_t, d_s, seed):
    """Overwrite ~2% of the samples with exact vertices of both lattices,
    0, 1, 1 - ulp and out-of-range values (the cell-selection edge cases)."""
    rng = np.random.default_rng(seed)
    rgb = rgb.copy()
    special = np.concatenate([np.arange(d_t) / np.float32(d_t - 1), np.arange(d_s) / np.float32(d_s - 1),
                              [0.0, 1.0, np.nextafter(np.float32(1), np.float32(0)), -0.25, 1.5,
                               np.float32(1e-30)]]).astype(np.float32)
    mask = rng.random(rgb.shape) < 0.02
    rgb[mask] = rng.choice(special, size=int(mask.sum()))
    return rgb


def lut_id_tables(d_t, d_s, batch):
    """Channel c's A coefficient of pair c's cell (i, j) = 1 + i*d_t + j."""
    L = Layout(d_t, d_s)
    t = empty_table(L)
    n = d_t - 1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ids = (1 + i * d_t + j).astype(np.float32)
    zero = np.zeros_like(ids)
    for pair in range(3):
        write_cells(t, L, pair, pair, np.stack([ids, zero, zero, zero]))
    return np.tile(t, batch)


def grid_id_tables(d_t, d_s, batch):
    """Merged xc cell (c, jx, jc) coefficient A = 1 + jx*d_s + jc (+ 1000 c)."""
    L = Layout(d_t, d_s)
    t = empty_table(L)
    n = d_s - 1
    jx, jc = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    for c in range(3):
        xc = t[L.xc_off:L.xc_off + 3 * n * n * 4].reshape(3, n, n, 4)
        xc[c, :, :, 0] = 1 + jx * d_s + jc + 1000 * c
    return np.tile(t, batch)


def run_ids(dev, table, rgb, d_t, d_s, y0=0, h_total=None):
    import torch

    from paper_2508_16121_b200 import device

    x = T(rgb, dev)
    if x.dim() == 3:
        x = x[None]
    tables = device.PackedTables(T(table, dev), x.shape[0], d_t, d_s)
    out = device.apply(x, tables, y0=y0, h_total=h_total)
    torch.cuda.synchronize()
    return out.cpu().numpy()


CASES = [
    # (name, d_t, d_s, h, w, y0, h_total)
    ("config2 4K", 33, 17, 2160, 3840, 0, None),
    ("8K strip y0=2700", 33, 17, 540, 7680, 2700, 4320),
    ("17/8 1080p", 17, 8, 1080, 1920, 0, None),
    ("generic 9/5 strip", 9, 5, 301, 517, 123, 999),
]


@pytest.mark.parametrize("name,d_t,d_s,h,w,y0,h_total", CASES)
def test_fused_kernel_lut_cell_selection(dev, oracle_mod, name, d_t, d_s, h, w, y0, h_total):
    from paper_2508_16121_b200 import synth

    case = synth.make_case(7, h=h, w=w, d_t=d_t, d_s=d_s)
    rgb = with_vertex_hits(case.rgb, d_t, d_s, seed=h + w)
    got = run_ids(dev, lut_id_tables(d_t, d_s, 1), rgb, d_t, d_s, y0, h_total)[0]
    idx = oracle_mod.indices(rgb, d_t, d_s, y0=y0, h_total=h_total)  # (8, H, W)
    ir, ig, ib = idx[0], idx[1], idx[2]
    for c, (a, b) in enumerate(((ir, ig), (ir, ib), (ig, ib))):
        want = (1 + a * d_t + b).astype(np.float32)
        bad = got[c] != want
        assert not bad.any(), (name, "pair", c, int(bad.sum()), np.argwhere(bad)[:3])


@pytest.mark.parametrize("name,d_t,d_s,h,w,y0,h_total", CASES)
def test_fused_kernel_grid_cell_selection(dev, oracle_mod, name, d_t, d_s, h, w, y0, h_total):
    from paper_2508_16121_b200 import synth

    case = synth.make_case(8, h=h, w=w, d_t=d_t, d_s=d_s)
    rgb = with_vertex_hits(case.rgb, d_t, d_s, seed=3 * h + w)
    got = run_ids(dev, grid_id_tables(d_t, d_s, 1), rgb, d_t, d_s, y0, h_total)[0]
    idx = oracle_mod.indices(rgb, d_t, d_s, y0=y0, h_total=h_total)
    jx = idx[6]
    for c in range(3):
        want = (1 + jx * d_s + idx[3 + c] + 1000 * c).astype(np.float32)
        bad = got[c] != want
        assert not bad.any(), (name, "channel", c, int(bad.sum()), np.argwhere(bad)[:3])


def oracle_fwd(oracle_mod, case, planes, rgb=None, **kw):
    return oracle_mod.fused_fwd(case.rgb if rgb is None else rgb, planes, case.lw, case.lb, case.grid_planes,
                                case.gw, case.gb, threads=oracle_mod.max_threads(), **kw)


def test_config3_sixteen_4k_images(dev, oracle_mod):
    """Config 3 at full size: 16 x 4K, each image with its own factors/grids,
    through the batched product path (factors -> tables -> fused apply)."""
    import torch

    from paper_2508_16121_b200 import device, synth

    for lo in range(0, 16, 4):
        cases = [synth.make_case(s) for s in range(lo, lo + 4)]
        st = {k: T(np.stack([getattr(c, k) for c in cases]), dev)
              for k in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
        tables = device.pack_tables_factors(st["u"], st["s"], st["vt"], st["lw"], st["lb"], st["grid_planes"],
                                            st["gw"], st["gb"])
        out = device.apply(st["rgb"], tables)
        torch.cuda.synchronize()
        for i, c in enumerate(cases):
            want = oracle_fwd(oracle_mod, c, oracle_mod.reconstruct(c.u, c.s, c.vt))
            err = float(np.abs(out[i].cpu().numpy() - want).max())
            assert err <= TOL, (lo + i, err)


def test_config4_8k_strips(dev, oracle_mod):
    """Config 4 at full size: 3x4320x7680 in 8 strips of 540 rows with
    (y0, H_total): bitwise equal to the unsplit run, which is within 1e-5 of
    the oracle."""
    import torch

    from paper_2508_16121_b200 import device, parallel, synth

    case = synth.make_case(0, h=4320, w=7680)
    p = {k: T(getattr(case, k), dev) for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    tables = device.pack_tables_factors(p["u"], p["s"], p["vt"], p["lw"], p["lb"], p["grid_planes"], p["gw"],
                                        p["gb"])
    x = T(case.rgb, dev)[None]
    full = device.apply(x, tables)
    parts = []
    for r in range(8):
        y0, y1 = parallel.strip_rows(4320, 8, r)
        assert y1 - y0 == 540
        parts.append(device.apply(x[:, :, y0:y1].contiguous(), tables, y0=y0, h_total=4320))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, dim=2), full)
    want = oracle_fwd(oracle_mod, case, oracle_mod.reconstruct(case.u, case.s, case.vt))
    assert float(np.abs(full[0].cpu().numpy() - want).max()) <= TOL


def rel_err(got, want):
    scale = max(float(np.abs(want).max()), 1e-30)
    return float(np.abs(np.asarray(got, np.float64) - want).max()) / scale


def test_config5_training_step_8x1080p(dev, oracle_mod):
    """Config 5 at full size: autograd.l2_step (fused loss epilogue, packed
    backward) on 8 x 1080p vs the f64 oracle backward + reconstruct backward,
    1e-4 relative per tensor (max |g - g_ref| <= 1e-4 max |g_ref|)."""
    import torch

    from paper_2508_16121_b200 import autograd, synth

    case = synth.make_batch(list(range(8)), h=1080, w=1920)
    st = {k: T(getattr(case, k), dev) for k in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    target = st["rgb"].clamp_min(0) ** 0.8
    g = autograd.l2_step(st["rgb"], target, st["u"], st["s"], st["vt"], st["lw"], st["lb"], st["grid_planes"],
                         st["gw"], st["gb"])
    torch.cuda.synchronize()
    tgt = target.cpu().numpy()
    n = case.rgb.size
    loss = 0.0
    for i in range(8):
        planes = oracle_mod.reconstruct(case.u[i], case.s[i], case.vt[i])
        y = oracle_mod.fused_fwd(case.rgb[i], planes, case.lw[i], case.lb[i], case.grid_planes[i], case.gw[i],
                                 case.gb[i], threads=oracle_mod.max_threads())
        r = y.astype(np.float64) - tgt[i]
        loss += float((r * r).sum())
        gy = (2.0 * r / n).astype(np.float32)
        ref = oracle_mod.fused_bwd(case.rgb[i], gy, planes, case.lw[i], case.grid_planes[i], case.gw[i])
        du, ds, dvt = oracle_mod.reconstruct_bwd(case.u[i], case.s[i], case.vt[i], ref["dlp"])
        pairs = {"gx": ref["gx"], "u": du, "s": ds, "vt": dvt, "lw": ref["dlw"], "lb": ref["dlb"],
                 "grid_planes": ref["dgp"], "gw": ref["dgw"], "gb": ref["dgb"]}
        for k, want in pairs.items():
            e = rel_err(g[k][i].cpu().numpy(), want)
            assert e <= 1e-4, (i, k, e)
    assert abs(float(g["loss"]) - loss / n) <= 1e-5 * (loss / n)
