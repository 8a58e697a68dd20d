"""Training path: the fused apply as a torch.autograd.Function (config 5).

    y = svdlut_apply(rgb, u, s, vt, lw, lb, grid_planes, gw, gb)
    loss = ((y - target) ** 2).mean(); loss.backward()

Forward: LUT reconstruction from the SVD factors + table packing + the fused
sm_100a kernel.  Backward: svdlut_fused_bwd (input gradient and
warp-aggregated shared-memory scatter of the LUT / grid vertex gradients) and
svdlut_reconstruct_bwd (dU, dS, dVt).  Gradient conventions at cell
boundaries and the clamp follow SURVEY.md Appendix B (the reference itself
has no backward).  Accepts batched (B, ...) or unbatched tensors.
"""

import torch

from . import device

__all__ = ["SvdLutApply", "svdlut_apply", "l2_step"]


class SvdLutApply(torch.autograd.Function):
    @staticmethod
    def forward(ctx, rgb, u, s, vt, lw, lb, grid_planes, gw, gb, y0=0, h_total=None):
        batched = rgb.dim() == 4
        planes = device.reconstruct(u, s, vt)
        if device.fast_supported(planes.shape[-1], grid_planes.shape[-1]):
            tables = device.pack_tables(planes, lw, lb, grid_planes, gw, gb)
            out = device.apply(rgb, tables, y0=y0, h_total=h_total)
        else:
            out = device.apply_exact(rgb, planes, lw, lb, grid_planes, gw, gb, y0=y0,
                                     h_total=h_total)
        ctx.save_for_backward(rgb, u, s, vt, planes, lw, grid_planes, gw)
        ctx.y0, ctx.h_total, ctx.batched = y0, h_total, batched
        ctx.shapes = [t.shape for t in (rgb, u, s, vt, lw, lb, grid_planes, gw, gb)]
        return out if batched else out[0]

    @staticmethod
    def backward(ctx, gy):
        rgb, u, s, vt, planes, lw, grid_planes, gw = ctx.saved_tensors
        gy = gy.contiguous()
        g = device.fused_backward(rgb, gy, planes, lw, grid_planes, gw, y0=ctx.y0,
                                  h_total=ctx.h_total, need_gx=ctx.needs_input_grad[0])
        du, ds, dvt = device.reconstruct_backward(u, s, vt, g["dlut_planes"])
        grads = [g["gx"], du, ds, dvt, g["dlw"], g["dlb"], g["dgrid_planes"], g["dgw"], g["dgb"]]
        out = []
        for gr, shape, need in zip(grads, ctx.shapes, ctx.needs_input_grad[:9]):
            out.append(gr.reshape(shape) if (need and gr is not None) else None)
        return (*out, None, None)


def svdlut_apply(rgb, u, s, vt, lw, lb, grid_planes, gw, gb, y0=0, h_total=None):
    return SvdLutApply.apply(rgb, u, s, vt, lw, lb, grid_planes, gw, gb, y0, h_total)


def l2_step(rgb, target, u, s, vt, lw, lb, grid_planes, gw, gb, need_gx=True, fused=True):
    """One training step of mean((Y - target)^2) without autograd overhead
    (BASELINE config 5): tables from the factors, then the pixel work in one
    pass (``fused=True``, svdlut_fused_l2_step: Y, the loss and gY are formed
    per pixel and feed the backward directly, so neither Y nor gY touches
    HBM), or as two kernels (``fused=False``: the forward with the loss fused
    into its epilogue writes gY and max|gY|, the backward reads them), and
    the factor gradients.  Returns a dict with the scalar ``loss`` (float64
    tensor) and the gradients keyed like SvdLutApply's inputs.
    """
    planes = device.reconstruct(u, s, vt)
    tables = device.pack_tables(planes, lw, lb, grid_planes, gw, gb)
    gscale = 2.0 / rgb.numel()
    if fused:
        loss_sum, g = device.fused_l2_step(rgb, target, tables, planes, lw, grid_planes, gw, gscale=gscale,
                                           need_gx=need_gx)
    else:
        gy, loss_sum, gmax = device.apply_l2(rgb, target, tables, gscale=gscale)
        # sum gY^2 per image = gscale^2 * sum (Y - T)^2: sets the scatter's
        # fixed-point bound (outlier residuals take the f32 path)
        g = device.fused_backward(rgb, gy, planes, lw, grid_planes, gw, need_gx=need_gx, tables=tables,
                                  gmax=gmax, gsumsq=loss_sum * (gscale * gscale))
    du, ds, dvt = device.reconstruct_backward(u, s, vt, g["dlut_planes"])
    return {"loss": loss_sum.sum() / rgb.numel(), "gx": g["gx"], "u": du, "s": ds, "vt": dvt,
            "lw": g["dlw"], "lb": g["dlb"], "grid_planes": g["dgrid_planes"], "gw": g["dgw"],
            "gb": g["dgb"]}
