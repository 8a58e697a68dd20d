"""CPU oracle (test infrastructure only) for the multi-pass "original
structure" and the 3D-LUT baseline: a numpy restatement of the reference's
stage functions, checked against outputs of the reference itself
(tests/golden/naive_golden.npz, tests/golden/make_naive_golden.py).

    bracket_array   interp.py:114-123   f32 product, f64 delta
    slice_grids     transform.py:144-178 (spatial brackets + slice_grid2d)
    apply_lut2d     transform.py:123-141
    combine_slices  transform.py:181-193
    apply_lut3d     transform.py:93-120
    naive_enhance   transform.py:196-212

Never imported by the product package.
"""

import numpy as np


def bracket_array(p, d):
    t = np.clip(p, 0.0, 1.0).astype(np.float32, copy=False) * np.float32(d - 1)
    i = np.minimum(np.floor(t), d - 2).astype(np.int32)
    return i, t - i  # float32 - int32 -> float64 (exact)


def _blend(plane, ia, da, ib, db):
    # four corners, f64 products, summed in this order
    out = plane[ia, ib] * ((1 - da) * (1 - db))
    out = out + plane[ia + 1, ib] * (da * (1 - db))
    out = out + plane[ia, ib + 1] * ((1 - da) * db)
    return out + plane[ia + 1, ib + 1] * (da * db)


def spatial_brackets(w, h, d, y0=0, h_total=None):
    h_total = h if h_total is None else h_total
    xs = np.arange(w, dtype=np.float32) / np.float32(w - 1)
    ys = np.arange(y0, y0 + h, dtype=np.float32) / np.float32(h_total - 1)
    return bracket_array(xs, d) + bracket_array(ys, d)


def slice_grids(rgb, gp, gw, gb, y0=0, h_total=None):
    """(K, H, W) float32 slicing maps."""
    _, h, w = rgb.shape
    k, d = gp.shape[0], gp.shape[-1]
    ix, dx, iy, dy = spatial_brackets(w, h, d, y0, h_total)
    ixb, dxb = np.broadcast_to(ix[None, :], (h, w)), np.broadcast_to(dx[None, :], (h, w))
    iyb, dyb = np.broadcast_to(iy[:, None], (h, w)), np.broadcast_to(dy[:, None], (h, w))
    guides = [bracket_array(rgb[c], d) for c in range(3)]
    fs = np.empty((k, h, w), np.float32)
    for kk in range(k):
        ic, dc = guides[kk % 3]
        acc = gw[kk, 0] * _blend(gp[kk, 0], ixb, dxb, iyb, dyb)
        acc = acc + gw[kk, 1] * _blend(gp[kk, 1], ixb, dxb, ic, dc)
        acc = acc + gw[kk, 2] * _blend(gp[kk, 2], iyb, dyb, ic, dc)
        fs[kk] = acc + gb[kk]
    return fs


def apply_lut2d(rgb, lp, lw, lb):
    d = lp.shape[-1]
    (ir, dr), (ig, dg), (ib, db) = (bracket_array(rgb[c], d) for c in range(3))
    out = np.empty(rgb.shape, np.float32)
    for c in range(3):
        acc = lw[c, 0] * _blend(lp[c, 0], ir, dr, ig, dg)
        acc = acc + lw[c, 1] * _blend(lp[c, 1], ir, dr, ib, db)
        acc = acc + lw[c, 2] * _blend(lp[c, 2], ig, dg, ib, db)
        out[c] = acc + lb[c]
    return out


def combine_slices(base, fs):
    out = np.empty(base.shape, np.float32)
    for c in range(3):
        s = fs[c].copy()
        for j in range(c + 3, fs.shape[0], 3):
            s += fs[j]  # float32, map order
        out[c] = base[c] + s
    return out


def naive_enhance(rgb, lp, lw, lb, gp, gw, gb):
    return combine_slices(apply_lut2d(rgb, lp, lw, lb), slice_grids(rgb, gp, gw, gb))


def apply_lut3d(rgb, cubes):
    d = cubes.shape[1]
    (ir, dr), (ig, dg), (ib, db) = (bracket_array(rgb[c], d) for c in range(3))
    out = np.empty(rgb.shape, np.float32)
    for c in range(3):
        cube = cubes[c]

        def slab(b):
            return _blend_rg(cube, ir, dr, ig, dg, b)

        out[c] = slab(ib) * (1 - db) + slab(ib + 1) * db
    return out


def _blend_rg(cube, ir, dr, ig, dg, ib):
    out = cube[ir, ig, ib] * ((1 - dr) * (1 - dg))
    out = out + cube[ir + 1, ig, ib] * (dr * (1 - dg))
    out = out + cube[ir, ig + 1, ib] * ((1 - dr) * dg)
    return out + cube[ir + 1, ig + 1, ib] * (dr * dg)


def occurrence(rgb, d):
    """analysis.occurrence_stats (analysis.py:109-122) for one image: int64 cube
    of bracketing-cell corner touches."""
    ir, ig, ib = (bracket_array(rgb[c], d)[0].astype(np.int64) for c in range(3))
    flat = np.zeros(d ** 3, np.int64)
    base = ((ir * d + ig) * d + ib).ravel()
    for corner in range(8):
        np.add.at(flat, base + ((corner >> 2) * d + ((corner >> 1) & 1)) * d + (corner & 1), 1)
    return flat.reshape(d, d, d)
