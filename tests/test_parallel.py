"""Multi-process (world size 2, gloo, CPU) tests of the sharding host logic.

Each rank computes its shard with the CPU oracle standing in for the kernel
(the oracle honours the same (y0, h_total) strip contract), gathers, and
checks the result against the unsplit oracle run bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_16121_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_apply(case):
    import oracle

    def fn(rgb, tables, y0, h_total):
        outs = []
        for b in range(rgb.shape[0]):
            t = tables[b]
            outs.append(torch.from_numpy(oracle.fused_fwd(
                rgb[b].numpy(), t["lp"], t["lw"], t["lb"], t["gp"], t["gw"], t["gb"], y0=y0,
                h_total=h_total)))
        return torch.stack(outs)
    return fn


def _make(seed, n_img, h, w):
    from conftest import make_inputs

    cases = [make_inputs(w, h, d_t=9, d_s=5, k=6, seed=seed + i) for i in range(n_img)]
    rgb = torch.from_numpy(np.stack([c["rgb"] for c in cases]))
    return rgb, cases


def _worker(rank, world, port, mode, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn = _oracle_apply(None)
        if mode == "strip":
            rgb, cases = _make(3, 1, 37, 29)
            y0, y1 = parallel.strip_rows(37, world, rank)
            mine = parallel.forward_strip(rgb[:, :, y0:y1], cases, y0, 37, apply_fn=fn)
            full = parallel.gather_rows(mine)
            want = fn(rgb, cases, 0, 37)
        else:
            rgb, cases = _make(7, 5, 11, 13)
            b0, b1 = parallel.image_block(5, world, rank)
            mine = parallel.forward_images(rgb[b0:b1], cases[b0:b1], apply_fn=fn)
            full = parallel.gather_images(mine)
            want = fn(rgb, cases, 0, 11)
        t = parallel.max_over_ranks(float(rank + 1))
        q.put((rank, bool(torch.equal(full, want)), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["strip", "image"])
def test_two_rank_sharding_matches_unsplit(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert all(t == 2.0 for _, _, t in res)  # max over ranks of (rank + 1)


def test_shard_ranges_partition_exactly():
    for n in (0, 1, 7, 2160, 4320):
        for world in (1, 2, 3, 4, 8):
            spans = [parallel.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_range(10, 2, 2)


def _torch_l2_step(rgb, target, batched):
    """CPU float64 stand-in for autograd.l2_step (tests/_torch_ref.py forward,
    planes from the factors, mean-square loss, autograd gradients)."""
    import _torch_ref

    t = {k: v.detach().clone().requires_grad_(True) for k, v in batched.items()}
    ys = []
    for b in range(rgb.shape[0]):
        planes = torch.matmul(t["u"][b] * t["s"][b][..., None, :], t["vt"][b])
        ys.append(_torch_ref.forward(rgb[b], planes, t["lw"][b], t["lb"][b], t["grid_planes"][b],
                                     t["gw"][b], t["gb"][b]))
    loss = ((torch.stack(ys) - target) ** 2).mean()
    loss.backward()
    out = {k: v.grad for k, v in t.items()}
    out["loss"] = loss.detach()
    return out


def _dp_inputs():
    rng = np.random.default_rng(11)
    d_t, n_s, d_s, k = 5, 3, 4, 6
    f = lambda *s: torch.from_numpy(rng.normal(0, 0.3, s))  # noqa: E731
    params = {"u": f(3, 3, d_t, n_s), "s": f(3, 3, n_s).abs(), "vt": f(3, 3, n_s, d_t),
              "lw": f(3, 3) + 1, "lb": f(3), "grid_planes": f(k, 3, d_s, d_s), "gw": f(k, 3) + 1,
              "gb": f(k)}
    rgb = torch.from_numpy(rng.random((3, 3, 9, 12)))
    target = rgb ** 0.8
    return rgb, target, params


def _dp_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rgb, target, params = _dp_inputs()
        b0, b1 = parallel.image_block(rgb.shape[0], world, rank)  # 2 + 1 images: unequal shards
        g = parallel.data_parallel_l2_step(rgb[b0:b1], target[b0:b1], params, step_fn=_torch_l2_step)
        q.put((rank, {k: v.numpy() for k, v in g.items()}))
    finally:
        dist.destroy_process_group()


def test_two_rank_shared_parameter_step_equals_full_batch():
    """One all_reduce(SUM) bucket turns per-rank gradients of a shared model
    into the gradient of the global mean loss (unequal shards)."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    rgb, target, params = _dp_inputs()
    want = parallel.data_parallel_l2_step(rgb, target, params, step_fn=_torch_l2_step)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got in res:
        for k, v in want.items():
            np.testing.assert_allclose(got[k], v.numpy(), rtol=1e-10, atol=1e-14, err_msg=k)
