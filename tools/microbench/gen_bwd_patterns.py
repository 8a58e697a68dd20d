"""Warp address patterns of the backward's LUT scatter and table gathers on
the synthetic smooth 1080p image, for atomspat.cu (word indices) and
ldsclean.cu (16-byte chunk indices), per lane -> pixel mapping:
  spread  lane l of warp w holds pixels 4(s0 + 15 l + w) + u (the kernel's)
  cons4   lane l holds pixels x0 + 4 l + u (the forward's)
  cons1   lane l holds pixel x0 + l + 32 u
Usage: python gen_bwd_patterns.py OUTDIR
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2508_16121_b200 import synth  # noqa: E402

out = sys.argv[1]
c = synth.make_case(0, h=1080, w=1920)
X = np.clip(c.rgb[0] if c.rgb.ndim == 4 else c.rgb, 0, 1)
dt, W = 33, 1920
idx = np.minimum(np.floor(X * (dt - 1)).astype(int), dt - 2)
rng = np.random.default_rng(0)
lanes = np.arange(32)


def pixels(mapping):
    y = int(rng.integers(0, 1080))
    u = int(rng.integers(0, 4))
    if mapping == "spread":
        w = int(rng.integers(0, 15))
        x = 4 * (lanes * 15 + w) + u
    elif mapping == "cons4":
        x0 = int(rng.integers(0, W // 128)) * 128
        x = x0 + 4 * lanes + u
    else:
        x0 = int(rng.integers(0, W // 128)) * 128
        x = x0 + lanes + 32 * u
    return y, np.minimum(x, W - 1)


with open(os.path.join(out, "atoms.txt"), "w") as fa, open(os.path.join(out, "lds.txt"), "w") as fl:
    for mapping in ("spread", "cons4", "cons1"):
        for rot in (0, 1):
            fa.write(f"# LUT rg corner00 {mapping} rot{rot}\n")
            for _ in range(48):
                y, x = pixels(mapping)
                base = (idx[0, y, x] * (dt + 1) + idx[1, y, x]) * 3
                fa.write(" ".join(str(v) for v in base + ((lanes % 3) if rot else 0)) + "\n")
        fl.write(f"# table rg chunk {mapping}\n")
        for _ in range(48):
            y, x = pixels(mapping)
            fl.write(" ".join(str(v) for v in idx[0, y, x] * 35 + idx[1, y, x]) + "\n")
    # corner x channel rotation (corner by (l / 3) % 4, channel by l % 3):
    # lanes sharing a cell hit twelve different words
    offs = np.array([0, (dt + 1) * 3, 3, (dt + 2) * 3])  # corners (0,0) (1,0) (0,1) (1,1)
    for mapping in ("spread", "cons4", "cons1"):
        fa.write(f"# LUT rg {mapping} rot12\n")
        for _ in range(48):
            y, x = pixels(mapping)
            base = (idx[0, y, x] * (dt + 1) + idx[1, y, x]) * 3
            k = int(rng.integers(0, 12))
            q = (k // 3 + lanes // 3) % 4
            cc = (k + lanes) % 3
            fa.write(" ".join(str(v) for v in base + offs[q] + cc) + "\n")
    # xc flush of the grid runs (channel 0): XR[jx][jc] + corner, d_s = 17
    ds = 17
    jcs = np.minimum(np.floor(X * (ds - 1)).astype(int), ds - 2)
    xoffs = np.array([0, ds, 1, ds + 1])
    for mapping in ("spread", "cons4"):
        for rot in (0, 1):
            fa.write(f"# grid xc {mapping} rot{rot}\n")
            for _ in range(48):
                y, x = pixels(mapping)
                jx = np.minimum(np.floor(x / (W - 1) * (ds - 1)).astype(int), ds - 2)
                q = (lanes % 4) if rot else np.zeros(32, int)
                fa.write(" ".join(str(v) for v in jx * ds + jcs[0, y, x] + xoffs[q]) + "\n")
    # synthetic sharing structures: k lanes per word, groups on random words
    for k in (1, 2, 4, 8, 16, 32):
        fa.write(f"# {k} lanes per word, random words\n")
        for _ in range(24):
            words = rng.integers(0, 4096, 32 // k)
            fa.write(" ".join(str(v) for v in np.repeat(words, k)) + "\n")
