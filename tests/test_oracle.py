"""Pin the CPU oracle to the real reference's outputs (golden vectors).

The oracle is the checker for every GPU parity test, so it must first agree
with the reference itself: bit-exact for the fused forward, cell selection
and spatial brackets; within 1 f32 ulp for reconstruct_lut (BLAS summation
order).  The backward oracle (no reference exists) is pinned against an
independent f64 torch autograd restatement and central finite differences.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden_case, make_inputs


def test_fused_forward_bit_exact_vs_reference(golden, oracle_mod):
    for name in golden["tr_cases"]:
        c = golden_case(golden, str(name))
        got = oracle_mod.fused_fwd(c["rgb"], c["lp"], c["lw"], c["lb"], c["gp"], c["gw"], c["gb"])
        assert np.array_equal(got, c["want"]), name


def test_fused_forward_thread_count_does_not_change_bits(golden, oracle_mod):
    c = golden_case(golden, "threads_64x48")
    a = oracle_mod.fused_fwd(c["rgb"], c["lp"], c["lw"], c["lb"], c["gp"], c["gw"], c["gb"], threads=1)
    b = oracle_mod.fused_fwd(c["rgb"], c["lp"], c["lw"], c["lb"], c["gp"], c["gw"], c["gb"], threads=7)
    assert np.array_equal(a, b) and np.array_equal(a, c["want"])


def test_straight_loop_agreement_matches_reference_tolerance(golden):
    # the reference pins fused vs its f64 loop oracle at 1e-5 (tests/test_transform.py:295)
    for name in golden["tr_cases"]:
        key = f"tr_{name}_loop"
        if key in golden:
            assert np.abs(golden[f"tr_{name}_want"] - golden[key]).max() <= 1e-5


def test_bracket_sweep_matches_reference(golden, oracle_mod):
    p = golden["br_p"]
    for d in golden["br_d"]:
        i, dl = oracle_mod.bracket_f64(p, int(d))
        assert np.array_equal(i, golden[f"br_{d}_i"]), d
        assert np.array_equal(dl, golden[f"br_{d}_d"]), d
        assert i.min() >= 0 and i.max() <= d - 2


def test_spatial_brackets_match_reference(golden, oracle_mod):
    for n, d in golden["sp_cases"]:
        ix, dx = oracle_mod.spatial(int(n), int(d))
        key = f"sp_{n}_{d}"
        if key + "_i" in golden:
            assert np.array_equal(ix, golden[key + "_i"]) and np.array_equal(dx, golden[key + "_d"])
        else:
            sha = hashlib.sha256(ix.tobytes() + dx.tobytes()).hexdigest()
            assert sha == str(golden[key + "_sha"]), (n, d)


def test_reconstruct_matches_reference(golden, oracle_mod):
    for i in golden["rc_cases"]:
        got = oracle_mod.reconstruct(golden[f"rc_{i}_u"], golden[f"rc_{i}_s"], golden[f"rc_{i}_vt"])
        want = golden[f"rc_{i}_planes"]
        ulp = np.spacing(np.abs(want).astype(np.float32))
        assert np.all(np.abs(got - want) <= ulp), i


def test_config1_end_to_end_bit_exact(golden, oracle_mod):
    """Reference run_model(720x480, seed 0) output reproduced from its tables."""
    rng = np.random.default_rng(0)
    rgb = rng.random((3, 480, 720), dtype=np.float32)
    assert hashlib.sha256(rgb.tobytes()).hexdigest() == str(golden["c1_input_sha"])
    planes = oracle_mod.reconstruct(golden["c1_u"], golden["c1_s"], golden["c1_vt"])
    assert np.array_equal(planes, golden["c1_planes"])
    y = oracle_mod.fused_fwd(rgb, planes, golden["c1_lw"], golden["c1_lb"], golden["c1_gp"],
                             golden["c1_gw"], golden["c1_gb"], threads=4)
    assert hashlib.sha256(y.tobytes()).hexdigest() == str(golden["c1_out_sha"])


def test_indices_match_bracket_definition(oracle_mod):
    inp = make_inputs(23, 17, d_t=7, d_s=8, seed=3, low=-0.3, high=1.3)
    idx = oracle_mod.indices(inp["rgb"], 7, 8)
    for c in range(3):
        i7, _ = oracle_mod.bracket_f64(inp["rgb"][c], 7)
        i8, _ = oracle_mod.bracket_f64(inp["rgb"][c], 8)
        assert np.array_equal(idx[c].ravel(), i7)
        assert np.array_equal(idx[3 + c].ravel(), i8)
    jx, _ = oracle_mod.spatial(23, 8)
    jy, _ = oracle_mod.spatial(17, 8)
    assert np.array_equal(idx[6], np.broadcast_to(jx[None, :], (17, 23)))
    assert np.array_equal(idx[7], np.broadcast_to(jy[:, None], (17, 23)))


def test_row_strips_bitwise_equal_unsplit(oracle_mod):
    inp = make_inputs(31, 29, d_t=9, d_s=5, seed=5)
    full = oracle_mod.fused_fwd(inp["rgb"], inp["lp"], inp["lw"], inp["lb"], inp["gp"], inp["gw"],
                                inp["gb"])
    parts = []
    for y0, y1 in ((0, 7), (7, 8), (8, 29)):
        parts.append(oracle_mod.fused_fwd(inp["rgb"][:, y0:y1], inp["lp"], inp["lw"], inp["lb"],
                                          inp["gp"], inp["gw"], inp["gb"], y0=y0, h_total=29))
    assert np.array_equal(np.concatenate(parts, axis=1), full)


@pytest.mark.parametrize("d_t,d_s,k", [(9, 5, 6), (7, 8, 9), (33, 17, 6)])
def test_backward_oracle_vs_torch_autograd(oracle_mod, d_t, d_s, k):
    import _torch_ref

    inp = make_inputs(11, 9, d_t=d_t, d_s=d_s, k=k, seed=d_t, low=-0.1, high=1.1)
    gy = np.random.default_rng(1).normal(size=(3, 9, 11)).astype(np.float32)
    g = oracle_mod.fused_bwd(inp["rgb"], gy, inp["lp"], inp["lw"], inp["gp"], inp["gw"])
    ref, y = _torch_ref.grads(inp, gy)
    yo = oracle_mod.fused_fwd(inp["rgb"], inp["lp"], inp["lw"], inp["lb"], inp["gp"], inp["gw"],
                              inp["gb"])
    assert np.abs(y - yo).max() <= 1e-5
    pairs = dict(gx="rgb", dlp="lp", dlw="lw", dlb="lb", dgp="gp", dgw="gw", dgb="gb")
    for mine, theirs in pairs.items():
        a, b = g[mine], ref[theirs]
        assert np.abs(a - b).max() <= 1e-9 * max(1.0, np.abs(b).max()), mine


def test_backward_oracle_vs_finite_differences(oracle_mod):
    import torch

    import _torch_ref

    inp = make_inputs(6, 5, d_t=9, d_s=5, seed=11, low=0.05, high=0.95)
    gy = np.random.default_rng(2).normal(size=(3, 5, 6))
    g = oracle_mod.fused_bwd(inp["rgb"], gy.astype(np.float32), inp["lp"], inp["lw"], inp["gp"],
                             inp["gw"])

    def loss(arrs):
        t = {k: torch.tensor(np.asarray(v, np.float64)) for k, v in arrs.items()}
        y = _torch_ref.forward(t["rgb"], t["lp"], t["lw"], t["lb"], t["gp"], t["gw"], t["gb"])
        return float((y.numpy() * gy).sum())

    rng = np.random.default_rng(3)
    eps = 1e-6
    for name, gname in (("rgb", "gx"), ("lp", "dlp"), ("gp", "dgp"), ("lw", "dlw"), ("gw", "dgw")):
        for _ in range(4):
            idx = tuple(int(rng.integers(0, s)) for s in inp[name].shape)
            plus = {k: np.array(v, np.float64) for k, v in inp.items()}
            minus = {k: np.array(v, np.float64) for k, v in inp.items()}
            plus[name][idx] += eps
            minus[name][idx] -= eps
            if name == "rgb":
                # stay inside one cell: skip queries too close to a vertex
                t = np.clip(inp["rgb"][idx], 0, 1) * np.array([8, 4])
                if np.any(np.abs(t - np.round(t)) < 1e-4):
                    continue
            fd = (loss(plus) - loss(minus)) / (2 * eps)
            assert abs(fd - g[gname][idx]) <= 1e-5 * max(1.0, abs(fd)), (name, idx)
