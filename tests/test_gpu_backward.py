"""GPU parity of the backward kernels against the f64 oracle (SURVEY.md
Appendix B; the reference itself has no backward — "parity unpinned" by the
reference, pinned by autograd + finite differences in test_oracle.py).
Tolerance (BASELINE.json north_star): 1e-4 relative, per tensor
max|g - g_ref| <= 1e-4 * max|g_ref|; touched-vertex pattern must match."""

import numpy as np
import pytest

from conftest import make_inputs

pytestmark = pytest.mark.gpu
RTOL = 1e-4


@pytest.fixture(scope="module")
def dev():
    import torch

    import __graft_entry__

    __graft_entry__.build_library()
    assert torch.cuda.is_available()
    return torch.device("cuda", 0)


def T(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def close(got, want, what):
    scale = max(float(np.abs(want).max()), 1e-30)
    err = float(np.abs(got - want).max())
    assert err <= RTOL * scale, f"{what}: err {err} vs scale {scale}"


@pytest.mark.parametrize("w,h,d_t,d_s,k,low,high", [
    (37, 21, 9, 5, 6, 0.0, 1.0),
    (64, 33, 33, 17, 6, -0.2, 1.2),
    (19, 40, 17, 8, 9, 0.0, 1.0),
    (5, 3, 2, 2, 3, -1.0, 2.0),
])
def test_fused_backward_vs_oracle(dev, oracle_mod, w, h, d_t, d_s, k, low, high):
    from paper_2508_16121_b200 import device

    c = make_inputs(w, h, d_t=d_t, d_s=d_s, k=k, seed=w + h, low=low, high=high)
    gy = np.random.default_rng(7).normal(size=(3, h, w)).astype(np.float32)
    g = device.fused_backward(T(c["rgb"], dev), T(gy, dev), T(c["lp"], dev), T(c["lw"], dev),
                              T(c["gp"], dev), T(c["gw"], dev))
    ref = oracle_mod.fused_bwd(c["rgb"], gy, c["lp"], c["lw"], c["gp"], c["gw"])
    names = dict(gx="gx", dlut_planes="dlp", dlw="dlw", dlb="dlb", dgrid_planes="dgp", dgw="dgw",
                 dgb="dgb")
    for mine, theirs in names.items():
        got = g[mine][0].cpu().numpy()
        close(got, ref[theirs], mine)
    # touched-vertex pattern: every vertex whose reference gradient exceeds the
    # tolerance is touched here too, and nothing untouched by the reference is
    # touched here (fixed-point accumulation may round sub-tolerance sums to 0)
    for mine, theirs in (("dlut_planes", "dlp"), ("dgrid_planes", "dgp")):
        got = g[mine][0].cpu().numpy()
        want = ref[theirs]
        big = np.abs(want) > RTOL * np.abs(want).max()
        assert np.all(got[big] != 0), mine
        assert np.all(got[want == 0] == 0), mine


def test_fused_backward_smooth_1080p_batch(dev, oracle_mod):
    """Config-5 shaped (smaller batch): smooth 1080p images, gY = 2(Y-T)/N."""
    import torch

    from paper_2508_16121_b200 import device, synth

    case = synth.make_batch([5, 6], h=1080, w=1920)
    t = {k: T(getattr(case, k), dev) for k in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes",
                                              "gw", "gb")}
    planes = device.reconstruct(t["u"], t["s"], t["vt"])
    y = device.fused_forward(t["rgb"], planes, t["lw"], t["lb"], t["grid_planes"], t["gw"], t["gb"])
    target = t["rgb"].clamp_min(0) ** 0.8
    gy = 2.0 * (y - target) / y.numel()
    g = device.fused_backward(t["rgb"], gy, planes, t["lw"], t["grid_planes"], t["gw"])
    for b in range(2):
        ref = oracle_mod.fused_bwd(case.rgb[b], gy[b].cpu().numpy(), planes[b].cpu().numpy(),
                                   case.lw[b], case.grid_planes[b], case.gw[b])
        close(g["gx"][b].cpu().numpy(), ref["gx"], "gx")
        close(g["dlut_planes"][b].cpu().numpy(), ref["dlp"], "dlut")
        close(g["dgrid_planes"][b].cpu().numpy(), ref["dgp"], "dgrid")
        close(g["dlw"][b].cpu().numpy(), ref["dlw"], "dlw")
        close(g["dgw"][b].cpu().numpy(), ref["dgw"], "dgw")
        close(g["dlb"][b].cpu().numpy(), ref["dlb"], "dlb")
        close(g["dgb"][b].cpu().numpy(), ref["dgb"], "dgb")
    torch.cuda.synchronize()


def test_reconstruct_backward_vs_oracle(dev, oracle_mod):
    from paper_2508_16121_b200 import device

    rng = np.random.default_rng(3)
    for d, n in ((33, 8), (9, 9), (2, 1)):
        u = rng.normal(0, 0.1, (3, 3, d, n)).astype(np.float32)
        s = rng.normal(0, 0.1, (3, 3, n)).astype(np.float32)
        vt = rng.normal(0, 0.1, (3, 3, n, d)).astype(np.float32)
        dT = rng.normal(size=(3, 3, d, d)).astype(np.float32)
        du, ds, dvt = device.reconstruct_backward(T(u, dev), T(s, dev), T(vt, dev), T(dT, dev))
        rdu, rds, rdvt = oracle_mod.reconstruct_bwd(u, s, vt, dT)
        close(du[0].cpu().numpy(), rdu, "du")
        close(ds[0].cpu().numpy(), rds, "ds")
        close(dvt[0].cpu().numpy(), rdvt, "dvt")


def test_autograd_matches_oracle_and_trains(dev, oracle_mod):
    """Config-5 style step through torch.autograd: L2 loss vs X^0.8."""
    import torch

    from paper_2508_16121_b200 import synth
    from paper_2508_16121_b200.autograd import svdlut_apply

    case = synth.make_batch([21, 22], h=72, w=128)
    leaves = {k: T(getattr(case, k), dev).requires_grad_(True)
              for k in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    rgb = T(case.rgb, dev).requires_grad_(True)
    target = (T(case.rgb, dev).clamp_min(0) ** 0.8).detach()
    y = svdlut_apply(rgb, leaves["u"], leaves["s"], leaves["vt"], leaves["lw"], leaves["lb"],
                     leaves["grid_planes"], leaves["gw"], leaves["gb"])
    loss = ((y - target) ** 2).mean()
    loss.backward()
    gy = (2.0 * (y - target) / y.numel()).detach()
    for b in range(2):
        planes = oracle_mod.reconstruct(case.u[b], case.s[b], case.vt[b])
        ref = oracle_mod.fused_bwd(case.rgb[b], gy[b].cpu().numpy(), planes, case.lw[b],
                                   case.grid_planes[b], case.gw[b])
        close(rgb.grad[b].cpu().numpy(), ref["gx"], "gx")
        close(leaves["grid_planes"].grad[b].cpu().numpy(), ref["dgp"], "dgrid")
        close(leaves["lw"].grad[b].cpu().numpy(), ref["dlw"], "dlw")
        du, ds_, dvt = oracle_mod.reconstruct_bwd(case.u[b], case.s[b], case.vt[b], ref["dlp"])
        close(leaves["u"].grad[b].cpu().numpy(), du, "du")
        close(leaves["s"].grad[b].cpu().numpy(), ds_, "ds")
        close(leaves["vt"].grad[b].cpu().numpy(), dvt, "dvt")
    # a few SGD steps on the tables decrease the loss
    opt = torch.optim.SGD(list(leaves.values()), lr=0.5)
    losses = []
    for _ in range(5):
        opt.zero_grad()
        y = svdlut_apply(rgb.detach(), leaves["u"], leaves["s"], leaves["vt"], leaves["lw"],
                         leaves["lb"], leaves["grid_planes"], leaves["gw"], leaves["gb"])
        l = ((y - target) ** 2).mean()
        l.backward()
        opt.step()
        losses.append(float(l))
    assert losses[-1] < losses[0]


def test_fused_l2_forward_epilogue(dev):
    """apply_l2: gy == (apply(x) - t) * 2/N (the epilogue's Y equals apply's up
    to the compiler's FMA contraction of the two instantiations: within 1e-6
    of max|gy|), gmax == max|gy| exactly, loss within 1e-6 relative of the
    f64 sum; the backward fed with the forward's tables (biases folded in, so
    float rounding of the biased grid vertices differs) and gmax matches the
    standalone backward within the gradient tolerance."""
    import torch

    from paper_2508_16121_b200 import device, synth

    cs = [synth.make_case(s, h=72, w=124) for s in (3, 4)]
    st = lambda f: T(np.stack([getattr(c, f) for c in cs]), dev)  # noqa: E731
    x = st("rgb")
    tgt = x.clamp_min(0) ** 0.8
    planes = device.reconstruct(st("u"), st("s"), st("vt"))
    tables = device.pack_tables(planes, st("lw"), st("lb"), st("grid_planes"), st("gw"), st("gb"))
    gy, loss, gmax = device.apply_l2(x, tgt, tables)
    y = device.apply(x, tables)
    scale = 2.0 / x.numel()
    ref = (y - tgt) * scale
    assert float((gy - ref).abs().max()) <= 1e-6 * float(ref.abs().max())
    assert torch.equal(gmax, gy.abs().flatten(1).max(dim=1).values)
    want = ((y.double() - tgt.double()) ** 2).flatten(1).sum(dim=1)
    assert float(((loss - want).abs() / want).max()) <= 1e-6
    g_ref = device.fused_backward(x, gy, planes, st("lw"), st("grid_planes"), st("gw"))
    g_pk = device.fused_backward(x, gy, planes, st("lw"), st("grid_planes"), st("gw"), tables=tables,
                                 gmax=gmax)
    for k in g_ref:
        close(g_pk[k].cpu().numpy(), g_ref[k].cpu().numpy(), k)


def test_l2_step_matches_autograd(dev):
    """autograd.l2_step (fused loss, no autograd graph) == SvdLutApply +
    torch loss + backward, gradients within the 1e-4 relative tolerance."""
    import torch

    from paper_2508_16121_b200 import autograd, synth

    c = synth.make_case(5, h=64, w=96)
    leaves = {f: T(getattr(c, f), dev)[None].requires_grad_(True)
              for f in ("rgb", "u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")}
    tgt = leaves["rgb"].detach().clamp_min(0) ** 0.8
    y = autograd.svdlut_apply(*leaves.values())
    loss = ((y - tgt) ** 2).mean()
    loss.backward()
    params = [leaves[f].detach() for f in ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")]
    step = autograd.l2_step(leaves["rgb"].detach(), tgt, *params)
    assert abs(float(step["loss"]) - float(loss)) <= 1e-6 * float(loss)
    names = {"rgb": "gx", "u": "u", "s": "s", "vt": "vt", "lw": "lw", "lb": "lb",
             "grid_planes": "grid_planes", "gw": "gw", "gb": "gb"}
    for leaf, key in names.items():
        close(step[key].reshape(leaves[leaf].grad.shape).cpu().numpy(),
              leaves[leaf].grad.cpu().numpy(), key)


def test_shared_parameter_step_matches_autograd(dev):
    """parallel.data_parallel_l2_step (single process: no exchange) on the
    kernels == autograd through SvdLutApply with ONE parameter set shared by
    a batch of 3 images."""
    import torch

    from paper_2508_16121_b200 import autograd, parallel, synth

    c = synth.make_case(8, h=40, w=72)
    rng = np.random.default_rng(8)
    rgb = T(rng.random((3, 3, 40, 72), dtype=np.float32), dev)
    tgt = rgb.clamp_min(0) ** 0.8
    params = {k: T(getattr(c, k), dev) for k in parallel.PARAM_KEYS}
    got = parallel.data_parallel_l2_step(rgb, tgt, params)
    leaves = {k: v.clone().requires_grad_(True) for k, v in params.items()}
    y = autograd.svdlut_apply(rgb, *(leaves[k].unsqueeze(0).expand(3, *leaves[k].shape).contiguous()
                                     for k in parallel.PARAM_KEYS))
    loss = ((y - tgt) ** 2).mean()
    loss.backward()
    assert abs(float(got["loss"]) - float(loss)) <= 1e-6 * float(loss)
    for k in parallel.PARAM_KEYS:
        close(got[k].cpu().numpy(), leaves[k].grad.cpu().numpy(), k)


def test_heavy_tailed_gy_keeps_small_contributions(dev, oracle_mod):
    """The scatter accumulates fixed point scaled by the image's max |gY|; a
    few outlier pixels 1e3x the rest must not wipe out the gradient the other
    pixels carry.  Checked per touched vertex against a RELATIVE tolerance on
    the vertices the small-residual pixels dominate."""
    from paper_2508_16121_b200 import device

    h, w = 96, 160
    c = make_inputs(w, h, d_t=33, d_s=17, k=6, seed=5)
    rng = np.random.default_rng(11)
    gy = rng.normal(size=(3, h, w)).astype(np.float32) * 1e-3
    out = rng.integers(0, h * w, 4)
    for o in out:  # four outliers, 1e3 x the typical residual
        gy[:, o // w, o % w] = 1.0
    g = device.fused_backward(T(c["rgb"], dev), T(gy, dev), T(c["lp"], dev), T(c["lw"], dev),
                              T(c["gp"], dev), T(c["gw"], dev))
    ref = oracle_mod.fused_bwd(c["rgb"], gy, c["lp"], c["lw"], c["gp"], c["gw"])
    for mine, theirs in (("dlut_planes", "dlp"), ("dgrid_planes", "dgp"), ("gx", "gx")):
        got = g[mine][0].cpu().numpy().astype(np.float64)
        want = ref[theirs]
        close(got, want, mine)
        # vertices whose reference gradient is at least 1e-2 of the tensor's
        # max (mostly carried by the small pixels): 1e-2 relative each
        big = np.abs(want) >= 1e-2 * np.abs(want).max()
        rel = np.abs(got[big] - want[big]) / np.abs(want[big])
        assert rel.max() <= 1e-2, (mine, float(rel.max()))


@pytest.mark.parametrize("b,h,w", [(3, 64, 200), (3, 400, 96)])
def test_backward_probe_bound_across_images_and_growth(dev, oracle_mod, b, h, w):
    """Without caller statistics each CTA takes its fixed-point bound from a
    probe of its first row and raises it on demand: a batch whose CTA row
    ranges cross image boundaries (1-2 and ~8 rows per CTA), with gY growing
    1e3x down each image (rescales inside a segment), still matches the f64
    oracle per image."""
    import torch

    from paper_2508_16121_b200 import device

    cs = [make_inputs(w, h, d_t=33, d_s=17, k=6, seed=40 + i) for i in range(b)]
    rng = np.random.default_rng(41)
    ramp = np.logspace(-3, 0, h, dtype=np.float32)[None, :, None]
    # mostly one sign (gradient sums that do not cancel: zero-mean noise sums
    # to ~sqrt(N) contributions, where any 2^-16 fixed-point step is ~1e-4)
    gys = [((1.0 + 0.3 * rng.normal(size=(3, h, w))) * ramp).astype(np.float32) for _ in range(b)]
    st = lambda key: T(np.stack([c[key] for c in cs]), dev)  # noqa: E731
    g = device.fused_backward(st("rgb"), T(np.stack(gys), dev), st("lp"), st("lw"), st("gp"), st("gw"))
    torch.cuda.synchronize()
    names = dict(gx="gx", dlut_planes="dlp", dlw="dlw", dlb="dlb", dgrid_planes="dgp", dgw="dgw", dgb="dgb")
    for i in range(b):
        ref = oracle_mod.fused_bwd(cs[i]["rgb"], gys[i], cs[i]["lp"], cs[i]["lw"], cs[i]["gp"], cs[i]["gw"])
        for mine, theirs in names.items():
            close(g[mine][i].cpu().numpy(), ref[theirs], f"{mine}[{i}]")
