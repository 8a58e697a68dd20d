"""Golden vectors for the generator path (paper_2508_16121_b200/network.py).

Run in the build container, where the reference package is importable:

    python tests/golden/make_network_golden.py [/root/reference]

Writes tests/golden/network_golden.npz:
  init_<seed>_<hyper>_sha   sha256 of every random_init tensor (canonical order)
  sm_*                      a small hyperparameter set on a 300x200 input
                            (upsampling resize): context, head outputs, and the
                            reference run_model output (sub-sampled + sha)
The default-hyperparameter config-1 vectors live in golden.npz (c1_*).
"""

import hashlib
import os
import sys

import numpy as np

SMALL = dict(m=4, d_t=17, d_s=9, k=3, n_s=4, m_s=5, m_t=6, m_sw=3, m_tw=2)


def main(ref_root):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.path.insert(0, os.path.join(ref_root, "pkg", "src"))
    from svdlut import core_types, network

    out = {}
    for seed, hp, tag in ((0, core_types.HyperParams(), "default"),
                          (3, core_types.HyperParams(**SMALL), "small")):
        params = network.random_init(seed, hp)
        h = hashlib.sha256()
        for name in core_types.expected_shapes(hp):
            h.update(np.ascontiguousarray(params.tensors[name]).tobytes())
        out[f"init_{seed}_{tag}_sha"] = np.array(h.hexdigest())

    hp = core_types.HyperParams(**SMALL)
    params = network.random_init(3, hp)
    rng = np.random.default_rng(7)
    img = core_types.Image(300, 200, rng.random((3, 200, 300), dtype=np.float32))
    ctx = network.backbone_forward(img, params)
    grids, gw, lut_factors, lw = network.generators_forward(ctx, params)
    y = network.run_model(img, params).data
    out.update({
        "sm_input_sha": np.array(hashlib.sha256(img.data.tobytes()).hexdigest()),
        "sm_ctx": ctx, "sm_u": lut_factors.u, "sm_s": lut_factors.s, "sm_vt": lut_factors.vt,
        "sm_lw": lw.w, "sm_lb": lw.b, "sm_gp": grids.planes, "sm_gw": gw.w, "sm_gb": gw.b,
        "sm_out_sub": y[:, ::3, ::5].copy(),
        "sm_out_sha": np.array(hashlib.sha256(y.tobytes()).hexdigest()),
    })
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "network_golden.npz")
    np.savez_compressed(dst, **out)
    print(f"wrote {dst}: {len(out)} arrays, {os.path.getsize(dst) / 1e6:.3f} MB")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference")
