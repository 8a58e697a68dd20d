"""Generate golden vectors from the REAL reference (run in the build container).

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py /root/reference

Imports the reference package (``pkg/src/svdlut``) and its own test helpers
(``pkg/tests/conftest.py`` generators, ``pkg/tests/reference.py`` straight-loop
oracle) and records inputs and outputs of the hot-path functions into
``tests/golden/golden.npz``.  The GPU box has no /root/reference; the tests
only read this file.  Cases follow the reference tests named in each key:

  tr_*   transform.fused_enhance on the reference's own test inputs
         (tests/test_transform.py:217-296) + defaults-dims / edge cases;
         ``want`` = reference fused output, ``loop`` = ref_enhance (f64 loop)
  rc_*   svd.reconstruct_lut (svd.py:210-220)
  br_*   interp._bracket sweep (interp.py:35-45, tests/test_interp.py:39-47)
  sp_*   transform._spatial_brackets (transform.py:144-149)
  c1_*   config 1: network.run_model on 720x480 seed 0 / random_init(0)
         (generator outputs, SHA-256 of the reference output, a subsample)
"""

import hashlib
import os
import sys

import numpy as np


def main(ref_root):
    sys.path[:0] = [os.path.join(ref_root, "pkg", "src"), os.path.join(ref_root, "pkg", "tests")]
    from conftest import (make_grid_weights, make_grids, make_image, make_lut2d,
                          make_lut_weights)
    from reference import ref_enhance
    from svdlut import interp, network, svd, transform
    from svdlut.core_types import GridSet, GridWeights, Image, Lut2DSet, LutWeights, SvdLut

    out = {}
    cases = []

    def add_case(name, img, luts, lw, grids, gw, loop=True):
        want = transform.fused_enhance(img, luts, lw, grids, gw).data
        rec = dict(rgb=img.data, lp=luts.planes, lw=lw.w, lb=lw.b, gp=grids.planes, gw=gw.w,
                   gb=gw.b, want=want)
        if loop:
            rec["loop"] = ref_enhance(img.data, luts.planes, lw.w, lw.b, grids.planes, gw.w, gw.b)
        for k, v in rec.items():
            out[f"tr_{name}_{k}"] = np.asarray(v)
        cases.append(name)

    # tests/test_transform.py:287-296 (fused & naive vs straight-loop oracle)
    add_case("match_reference", make_image(8, 8, seed=41), make_lut2d(d=7, seed=42),
             make_lut_weights(seed=43), make_grids(k=6, d=5, seed=44), make_grid_weights(k=6, seed=45))
    # :276-284
    add_case("fused_16x16", make_image(16, 16, seed=36), make_lut2d(d=9, seed=37),
             make_lut_weights(seed=38), make_grids(k=6, d=5, seed=39), make_grid_weights(k=6, seed=40))
    # :329-337 (thread-count test inputs)
    add_case("threads_64x48", make_image(64, 48, seed=48), make_lut2d(d=9, seed=49),
             make_lut_weights(seed=50), make_grids(k=6, d=5, seed=51),
             make_grid_weights(k=6, seed=52), loop=False)
    # :340-355 random trials (same rng stream as the reference test)
    rng = np.random.default_rng(53)
    for trial in range(10):
        w = int(rng.integers(2, 33))
        h = int(rng.integers(2, 33))
        d_t = int(rng.integers(2, 17))
        k = 3 * int(rng.integers(1, 4))
        d_s = int(rng.integers(2, 9))
        add_case(f"trial{trial}", make_image(w, h, seed=100 + trial),
                 make_lut2d(d=d_t, seed=200 + trial), make_lut_weights(seed=300 + trial),
                 make_grids(k=k, d=d_s, seed=400 + trial), make_grid_weights(k=k, seed=500 + trial),
                 loop=False)
    # default dims (d_t=33, d_s=17, K=6), out-of-range inputs
    add_case("defaults_97x61", make_image(97, 61, seed=7, low=-0.2, high=1.2),
             make_lut2d(d=33, seed=8), make_lut_weights(seed=9), make_grids(k=6, d=17, seed=10),
             make_grid_weights(k=6, seed=11), loop=False)
    # non power-of-two d-1 (exact-floor logic), K=9, tiny images
    add_case("d17_d8_k9", make_image(45, 31, seed=12), make_lut2d(d=17, seed=13),
             make_lut_weights(seed=14), make_grids(k=9, d=8, seed=15),
             make_grid_weights(k=9, seed=16), loop=False)
    add_case("d7_d7_k3", make_image(29, 23, seed=17, low=-0.5, high=1.5), make_lut2d(d=7, seed=18),
             make_lut_weights(seed=19), make_grids(k=3, d=7, seed=20),
             make_grid_weights(k=3, seed=21), loop=False)
    add_case("d2_d2_2x2", make_image(2, 2, seed=22), make_lut2d(d=2, seed=23),
             make_lut_weights(seed=24), make_grids(k=3, d=2, seed=25),
             make_grid_weights(k=3, seed=26))
    # exact vertex hits: 0, 1, k/(d-1), 1 - ulp, and just outside the range
    d_t, d_s = 33, 17
    vals = np.concatenate([
        np.array([0.0, 1.0, -0.0, -1e-7, 1.0 + 1e-7, 0.5, 0.25, np.nextafter(1.0, 0.0),
                  np.nextafter(0.0, 1.0), 2.0, -3.0], np.float32),
        (np.arange(33) / np.float32(32)).astype(np.float32),
        (np.arange(17) / np.float32(16)).astype(np.float32),
        (np.arange(7) / np.float32(6)).astype(np.float32),
        (np.arange(16) / np.float32(15)).astype(np.float32),
    ])
    vrng = np.random.default_rng(27)
    edge = vrng.permutation(np.resize(vals, 3 * 19 * 13)).reshape(3, 19, 13).astype(np.float32)
    add_case("vertex_hits", Image(13, 19, edge), make_lut2d(d=d_t, seed=28),
             make_lut_weights(seed=29), make_grids(k=6, d=d_s, seed=30),
             make_grid_weights(k=6, seed=31), loop=False)
    add_case("vertex_hits_d16", Image(13, 19, edge), make_lut2d(d=16, seed=32),
             make_lut_weights(seed=33), make_grids(k=6, d=7, seed=34),
             make_grid_weights(k=6, seed=35), loop=False)
    out["tr_cases"] = np.array(cases)

    # reconstruct_lut
    rrng = np.random.default_rng(61)
    rc = []
    for i, (d, n) in enumerate([(33, 8), (33, 33), (17, 4), (9, 1), (2, 2)]):
        u = rrng.normal(0, 0.1, (3, 3, d, n)).astype(np.float32)
        s = -np.sort(-rrng.normal(0, 0.1, (3, 3, n)), axis=-1).astype(np.float32)
        vt = rrng.normal(0, 0.1, (3, 3, n, d)).astype(np.float32)
        planes = svd.reconstruct_lut(SvdLut(u, s, vt)).planes
        out.update({f"rc_{i}_u": u, f"rc_{i}_s": s, f"rc_{i}_vt": vt, f"rc_{i}_planes": planes})
        rc.append(i)
    out["rc_cases"] = np.array(rc)

    # _bracket sweep (float32 queries, as the fused kernel feeds it)
    p = np.concatenate([np.linspace(-0.5, 1.5, 401), [0.0, 1.0, -0.0],
                        np.random.default_rng(62).uniform(-0.2, 1.2, 2000)]).astype(np.float32)
    p = np.concatenate([p, (np.arange(65) / np.float32(64)).astype(np.float32),
                        np.nextafter(np.float32(1.0), np.float32(0.0), dtype=np.float32)[None]])
    out["br_p"] = p
    ds_list = [2, 3, 5, 7, 9, 16, 17, 33, 64, 65]
    out["br_d"] = np.array(ds_list)
    for d in ds_list:
        idx = np.empty(p.size, np.int32)
        dl = np.empty(p.size, np.float64)
        for j, v in enumerate(p):
            i, e = interp._bracket(v, d)
            idx[j], dl[j] = i, e
        out[f"br_{d}_i"], out[f"br_{d}_d"] = idx, dl

    # spatial brackets
    sp = []
    for n in [2, 3, 7, 480, 720, 854, 1080, 1920, 2160, 3840, 4320, 7680]:
        for d in [2, 5, 8, 17, 33]:
            ix, dx, _, _ = transform._spatial_brackets(n, 2, d)
            key = f"sp_{n}_{d}"
            if n <= 854:
                out[key + "_i"], out[key + "_d"] = ix, dx
            else:
                out[key + "_sha"] = np.array(hashlib.sha256(ix.tobytes() + dx.tobytes()).hexdigest())
            sp.append((n, d))
    out["sp_cases"] = np.array(sp)

    # config 1 end to end: run_model(720x480, seed 0) with random_init(0)
    params = network.random_init(0)
    rng = np.random.default_rng(0)
    img = Image(720, 480, rng.random((3, 480, 720), dtype=np.float32))
    ctx = network.backbone_forward(img, params)
    grids, gw, lut_factors, lw = network.generators_forward(ctx, params)
    luts = svd.reconstruct_lut(lut_factors)
    y = network.run_model(img, params).data
    out.update({
        "c1_input_sha": np.array(hashlib.sha256(img.data.tobytes()).hexdigest()),
        "c1_ctx": ctx, "c1_u": lut_factors.u, "c1_s": lut_factors.s, "c1_vt": lut_factors.vt,
        "c1_lw": lw.w, "c1_lb": lw.b, "c1_gp": grids.planes, "c1_gw": gw.w, "c1_gb": gw.b,
        "c1_planes": luts.planes,
        "c1_out_sha": np.array(hashlib.sha256(y.tobytes()).hexdigest()),
        "c1_out_sub": y[:, ::7, ::11].copy(),
    })
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(dst, **out)
    print(f"wrote {dst}: {len(out)} arrays, {os.path.getsize(dst) / 1e6:.2f} MB")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference")
