"""Python mirror of the packed-table layout (paper_2508_16121_b200/csrc/svdlut_common.cuh).

Used by the boundary test (sizes) and by the poisoned-table GPU test, which
builds packed tables by hand so that the fused kernel's output reveals the
cell it selected.  Floats throughout.
"""

import numpy as np


def cst_for(dt):
    return (dt - 1) + ((3 - (dt - 1)) & 7)


class Layout:
    def __init__(self, dt, ds):
        self.dt, self.ds = dt, ds
        self.cst = cst_for(dt)
        self.tiles = (dt + 2) // 4
        self.plane_floats = max((dt - 1) * self.cst, self.tiles * self.tiles * 16) * 4
        self.lut_off = 0
        self.xc_off = self.lut_off + 9 * self.plane_floats
        self.gxy_off = self.xc_off + 3 * (ds - 1) * (ds - 1) * 4
        self.gyc_off = self.gxy_off + ((ds * ds * 3 + 3) & ~3)
        self.total_floats = (self.gyc_off + 3 * ds * ds + 31) & ~31

    @property
    def bytes(self):
        return self.total_floats * 4

    def plane_off(self, p, k):
        return self.lut_off + (3 * p + k) * self.plane_floats


def coef_slot(c, q):
    """Float position (0..11) of coefficient q (A, B, C, D) of channel c in a
    cell's three chunks {A0 A1 B0 B1} {C0 C1 D0 D1} {A2 C2 B2 D2}."""
    if c < 2:
        return (c, 2 + c, 4 + c, 6 + c)[q]
    return (8, 10, 9, 11)[q]


TILED_PLANES = {4, 5, 6, 7, 8}  # svdlut_common.cuh kTiledPlanes: rb chunks 1-2, gb chunks 0-2


def cell_index(L, idx, i, j):
    """Cell (i, j) within chunk plane idx = 3*pair + chunk: row stride cst, or
    4x4 tiles for the texture-path planes (svdlut_common.cuh)."""
    if idx not in TILED_PLANES:
        return i * L.cst + j
    return ((i >> 2) * L.tiles + (j >> 2)) * 16 + ((i & 3) << 2) + (j & 3)


def write_cells(table, L, p, c, coef):
    """Write coefficient arrays coef (4, dt-1, dt-1) = (A, B, C, D) of channel
    c, pair p (cells (i, j)), into a flat table."""
    n = L.dt - 1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    for q in range(4):
        slot = coef_slot(c, q)
        base = L.plane_off(p, slot // 4)
        plane = table[base:base + L.plane_floats].reshape(-1, 4)
        plane[cell_index(L, 3 * p + slot // 4, i, j), slot % 4] = coef[q]


def empty_table(L):
    return np.zeros(L.total_floats, np.float32)
