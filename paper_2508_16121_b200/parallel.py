"""Multi-GPU sharding of the apply path.

Every output pixel depends only on its own input pixel, its global (x, y) and
the per-image tables, so the path shards with no data-path exchange:

* per image  (configs 3 and 5): rank r takes a contiguous block of images;
* per strip  (config 4): rank r takes a contiguous block of rows of one image
  and evaluates it with ``(y0, h_total)`` so positions are normalised by the
  global height — the strips are bitwise equal to the unsplit run.

Tables (≈180 KB per image) are replicated.  NCCL is used only outside the
timed region: max-over-ranks timings and (optionally) gathering outputs for a
parity check.  ``apply_fn`` is injectable so the host logic is tested on CPU
with ``gloo`` (tests/test_parallel.py); the default runs the sm_100a kernels.
"""

import torch
import torch.distributed as dist

__all__ = ["shard_range", "strip_rows", "image_block", "forward_strip", "forward_images",
           "gather_rows", "gather_images", "max_over_ranks", "data_parallel_l2_step", "PARAM_KEYS"]

# parameter set of one SvdLut model, in autograd.l2_step's argument order
PARAM_KEYS = ("u", "s", "vt", "lw", "lb", "grid_planes", "gw", "gb")


def shard_range(n, world, rank):
    """Contiguous [lo, hi) share of n units for rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return n * rank // world, n * (rank + 1) // world


def strip_rows(h_total, world, rank):
    return shard_range(h_total, world, rank)


def image_block(batch, world, rank):
    return shard_range(batch, world, rank)


def _device_apply(rgb, tables, y0, h_total):
    from . import device

    return device.apply(rgb, tables, y0=y0, h_total=h_total)


def forward_strip(rgb_strip, tables, y0, h_total, apply_fn=None):
    """Apply to rows [y0, y0 + H_strip) of an image with h_total rows."""
    fn = apply_fn or _device_apply
    return fn(rgb_strip, tables, y0, h_total)


def forward_images(rgb_block, tables_block, apply_fn=None):
    """Apply to this rank's block of whole images (each with its own tables)."""
    fn = apply_fn or _device_apply
    return fn(rgb_block, tables_block, 0, rgb_block.shape[-2])


def _pad_gather(t, world, group, dim):
    """all_gather of tensors whose size along `dim` differs by at most one."""
    n = torch.tensor([t.shape[dim]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    if t.shape[dim] < m:
        pad_shape = list(t.shape)
        pad_shape[dim] = m - t.shape[dim]
        t = torch.cat([t, t.new_zeros(pad_shape)], dim=dim)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t.contiguous(), group=group)
    return torch.cat([b.narrow(dim, 0, s) for b, s in zip(bufs, sizes)], dim=dim)


def gather_rows(strip, group=None):
    """Concatenate every rank's (..., 3, rows, W) strip along the row axis."""
    world = dist.get_world_size(group)
    return _pad_gather(strip, world, group, dim=-2)


def gather_images(block, group=None):
    """Concatenate every rank's (B_r, 3, H, W) block along the batch axis."""
    world = dist.get_world_size(group)
    return _pad_gather(block, world, group, dim=0)


def max_over_ranks(value, device=None, group=None):
    """Max of a per-rank scalar (timing) — the only collective on the path."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def _device_l2_step(rgb, target, batched):
    from . import autograd

    return autograd.l2_step(rgb, target, *(batched[k] for k in PARAM_KEYS), need_gx=False)


def data_parallel_l2_step(rgb, target, params, group=None, step_fn=None):
    """One data-parallel training step of ONE shared parameter set.

    The per-image path (configs 3 / 5) needs no exchange; when a single model
    (unbatched ``params``: u, s, vt, lw, lb, grid_planes, gw, gb) is trained on
    a batch sharded over ranks, the table gradients are the one real exchange
    (SURVEY §8e).  Each rank runs the fused L2 step on its images with the
    parameters broadcast per image, sums the per-image gradients, converts
    them to the sum-of-squares form (x local pixel count) and issues ONE
    all_reduce(SUM) over a single flat bucket (≈80 KB at d_t=33 / d_s=17,
    latency-bound, so one bucket beats overlap) that also carries the loss
    sum and the pixel count; dividing by the global count gives every rank
    the gradient of the global mean((Y - target)^2).

    Returns {"loss": float tensor, key: gradient shaped like params[key]}.
    ``step_fn(rgb, target, batched_params)`` defaults to autograd.l2_step on
    the sm_100a kernels; tests inject a CPU stand-in (gloo).
    """
    fn = step_fn or _device_l2_step
    b = rgb.shape[0]
    batched = {k: params[k].unsqueeze(0).expand(b, *params[k].shape).contiguous() for k in PARAM_KEYS}
    g = fn(rgb, target, batched)
    n_local = float(rgb.numel())
    parts = [g[k].sum(0).reshape(-1).to(torch.float64) * n_local for k in PARAM_KEYS]
    loss = torch.as_tensor(g["loss"], dtype=torch.float64, device=parts[0].device).reshape(1)
    flat = torch.cat(parts + [loss * n_local, torch.tensor([n_local], dtype=torch.float64,
                                                           device=parts[0].device)])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    n_global = flat[-1]
    out, off = {}, 0
    for k in PARAM_KEYS:
        n = params[k].numel()
        out[k] = (flat[off:off + n] / n_global).reshape(params[k].shape).to(params[k].dtype)
        off += n
    out["loss"] = flat[off] / n_global
    return out
