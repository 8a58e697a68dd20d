"""float64 torch (CPU) autograd restatement of the fused apply — test infrastructure.

Independent route for the backward: the forward is
written from reference tests/reference.py:117-128 (ref_enhance) with integer
cell indices taken from the oracle (detached) and differentiable deltas
delta = clamp(X,0,1)*(d-1) - i, so autograd yields the reference-convention
gradients (torch.clamp passes the gradient for 0 <= X <= 1, matching the
strict clamp of interp.py:37-40).
"""

import numpy as np
import torch

import oracle


def _bil(P, ia, da, ib, db):
    return ((1 - da) * (1 - db) * P[ia, ib] + da * (1 - db) * P[ia + 1, ib]
            + (1 - da) * db * P[ia, ib + 1] + da * db * P[ia + 1, ib + 1])


def forward(rgb, lp, lw, lb, gp, gw, gb, y0=0, h_total=None):
    """All arguments float64 torch tensors (unbatched); returns Y (3,H,W)."""
    _, h, w = rgb.shape
    h_total = h if h_total is None else h_total
    d_t, d_s, k = lp.shape[2], gp.shape[2], gp.shape[0]
    idx = torch.from_numpy(oracle.indices(rgb.detach().numpy().astype(np.float32), d_t, d_s, y0,
                                          h_total).astype(np.int64))
    q = torch.clamp(rgb, 0.0, 1.0)
    it, js = idx[0:3], idx[3:6]
    dt_ = q * (d_t - 1) - it
    ds_ = q * (d_s - 1) - js
    ix, dx = oracle.spatial(w, d_s)
    iy_all, dy_all = oracle.spatial(h_total, d_s)
    jx = torch.from_numpy(ix.astype(np.int64))[None, :].expand(h, w)
    ex = torch.from_numpy(dx)[None, :].expand(h, w)
    jy = torch.from_numpy(iy_all[y0:y0 + h].astype(np.int64))[:, None].expand(h, w)
    ey = torch.from_numpy(dy_all[y0:y0 + h])[:, None].expand(h, w)
    pairs = ((0, 1), (0, 2), (1, 2))
    outs = []
    for c in range(3):
        acc = lb[c] + 0.0 * rgb[0]
        for p, (a, b) in enumerate(pairs):
            acc = acc + lw[c, p] * _bil(lp[c, p], it[a], dt_[a], it[b], dt_[b])
        for kk in range(c, k, 3):
            acc = acc + gw[kk, 0] * _bil(gp[kk, 0], jx, ex, jy, ey)
            acc = acc + gw[kk, 1] * _bil(gp[kk, 1], jx, ex, js[c], ds_[c])
            acc = acc + gw[kk, 2] * _bil(gp[kk, 2], jy, ey, js[c], ds_[c])
            acc = acc + gb[kk]
        outs.append(acc)
    return torch.stack(outs)


def grads(inputs, gy, y0=0, h_total=None):
    """Autograd gradients for numpy inputs dict and cotangent gy (3,H,W)."""
    t = {k: torch.tensor(np.asarray(v, np.float64), requires_grad=True)
         for k, v in inputs.items()}
    y = forward(t["rgb"], t["lp"], t["lw"], t["lb"], t["gp"], t["gw"], t["gb"], y0, h_total)
    (y * torch.tensor(np.asarray(gy, np.float64))).sum().backward()
    return {k: v.grad.numpy() for k, v in t.items()}, y.detach().numpy()
