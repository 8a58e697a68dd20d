"""Parameter-generator path on the GPU.

Restates the reference's context backbone and generator heads
(reference network.py:82-186) in PyTorch on device, batched, so that the whole
image-adaptive pipeline — resize, backbone, four heads, LUT reconstruction
from the SVD factors, table packing and the fused apply — runs in HBM without
a host round trip:

    gen = Generator(params, device="cuda")
    y = gen.enhance(rgb)                      # (B, 3, H, W) CUDA tensor in and out
    y = run_model(img, params)                # reference-facing: Image in, Image out

The backbone is small (five 3x3 stride-2 convolutions on a 256x256 resize,
~0.1 GFLOP per image) and stays PyTorch/cuDNN by design (BASELINE north star);
TF32 is disabled inside every call so the convolutions and head GEMMs run in
full fp32 like the reference's numpy (the end-to-end tolerance is 1e-5).  The
hot path after the heads is the sm_100a library: ``svdlut_pack_tables_factors``
builds the packed tables straight from U, S, Vt and ``svdlut_fused_fwd_packed``
applies them.

Parameters use the reference's names, shapes and canonical order
(core_types.py:305-332); ``random_init`` draws them exactly like
network.py:69-79, so ``random_init(seed)`` here and in the reference produce
bit-identical tensors (tests/golden/network_golden.npz pins this).
"""

from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from .core_types import Image as _Image
from .errors import DimensionMismatch, InvalidArgument

__all__ = ["HyperParams", "ModelParams", "expected_shapes", "random_init", "param_count",
           "Generator", "backbone_forward", "heads_forward", "run_model"]

_LEAKY_SLOPE = 0.2
_IN_EPS = 1e-5


@dataclass(frozen=True)
class HyperParams:
    """Architecture constants (reference core_types.py:259-286)."""

    m: int = 8
    d_t: int = 33
    d_s: int = 17
    k: int = 6
    n_s: int = 8
    m_s: int = 8
    m_t: int = 8
    m_sw: int = 8
    m_tw: int = 8
    n_sw: int = 3
    n_sb: int = 1
    n_tw: int = 3
    n_tb: int = 1

    def __post_init__(self):
        # reference core_types.py:335-349
        if self.m < 1:
            raise InvalidArgument("m must be >= 1")
        if self.d_t < 2 or self.d_s < 2:
            raise InvalidArgument("d_t and d_s must be >= 2")
        if self.k < 3 or self.k % 3 != 0:
            raise InvalidArgument("k must be a positive multiple of 3")
        if not 1 <= self.n_s <= self.d_t:
            raise InvalidArgument(f"n_s must be in 1..{self.d_t}")
        for name in ("m_s", "m_t", "m_sw", "m_tw"):
            if getattr(self, name) < 1:
                raise InvalidArgument(f"{name} must be >= 1")
        if (self.n_sw, self.n_sb, self.n_tw, self.n_tb) != (3, 1, 3, 1):
            raise InvalidArgument("weight heads must emit 3 weights and 1 bias")

    @property
    def ctx_dim(self) -> int:
        return 32 * self.m


@dataclass(frozen=True)
class ModelParams:
    """Named weight tensors + hyperparameters (reference core_types.py:289-302)."""

    hyper: HyperParams
    tensors: dict

    def __post_init__(self):
        want = expected_shapes(self.hyper)
        for name, shape in want.items():
            if name not in self.tensors:
                raise DimensionMismatch(f"missing tensor {name}")
            if tuple(self.tensors[name].shape) != shape:
                raise DimensionMismatch(
                    f"tensor {name} has shape {tuple(self.tensors[name].shape)}, expected {shape}")
        for name in self.tensors:
            if name not in want:
                raise DimensionMismatch(f"unexpected tensor {name}")


def expected_shapes(hyper: HyperParams) -> "dict[str, tuple[int, ...]]":
    """Canonical name -> shape map; iteration order = storage/init order
    (reference core_types.py:305-332)."""
    m = hyper.m
    widths = (3, m, 2 * m, 4 * m, 8 * m, 8 * m)
    shapes = {}
    for i in range(1, 6):
        cin, cout = widths[i - 1], widths[i]
        shapes[f"backbone.conv{i}.weight"] = (cout, cin, 3, 3)
        shapes[f"backbone.conv{i}.bias"] = (cout,)
        if i <= 4:
            shapes[f"backbone.in{i}.scale"] = (cout,)
            shapes[f"backbone.in{i}.shift"] = (cout,)
    ctx = hyper.ctx_dim
    heads = (
        ("grid_gen", hyper.m_s, hyper.k * 3 * hyper.d_s * hyper.d_s),
        ("gridw_gen", hyper.m_sw, hyper.k * (hyper.n_sw + hyper.n_sb)),
        ("lut_gen", hyper.m_t, 9 * (2 * hyper.d_t * hyper.n_s + hyper.n_s)),
        ("lutw_gen", hyper.m_tw, 3 * (hyper.n_tw + hyper.n_tb)),
    )
    for name, hidden, out in heads:
        shapes[f"{name}.fc1.weight"] = (hidden, ctx)
        shapes[f"{name}.fc1.bias"] = (hidden,)
        shapes[f"{name}.fc2.weight"] = (out, hidden)
        shapes[f"{name}.fc2.bias"] = (out,)
    return shapes


def param_count(hyper: HyperParams = HyperParams()) -> int:
    return sum(int(np.prod(s)) for s in expected_shapes(hyper).values())


def random_init(seed: int, hyper: HyperParams = HyperParams()) -> ModelParams:
    """U(-0.05, 0.05) float32 tensors drawn in canonical order from
    default_rng(seed) (reference network.py:69-79: bit-identical)."""
    rng = np.random.default_rng(seed)
    tensors = {name: rng.uniform(-0.05, 0.05, shape).astype(np.float32)
               for name, shape in expected_shapes(hyper).items()}
    return ModelParams(hyper, tensors)


@contextmanager
def _fp32_math():
    """Full-precision conv/GEMM (no TF32) for the duration of a call."""
    import torch

    saved = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = saved


def _hyper_of(params):
    h = params.hyper
    if isinstance(h, HyperParams):
        return h
    return HyperParams(**{f: getattr(h, f) for f in HyperParams.__dataclass_fields__})


class Generator:
    """Device-resident copy of a parameter set (ours or the reference's
    ModelParams: anything with ``.hyper`` and ``.tensors``)."""

    def __init__(self, params, device="cuda"):
        import torch

        self.hyper = _hyper_of(params)
        want = expected_shapes(self.hyper)
        self.device = torch.device(device)
        self.t = {}
        for name, shape in want.items():
            a = np.ascontiguousarray(params.tensors[name], dtype=np.float32)
            if a.shape != shape:
                raise DimensionMismatch(f"tensor {name} has shape {a.shape}, expected {shape}")
            self.t[name] = torch.from_numpy(a.copy()).to(self.device)

    # ---- reference network.py:82-128: resize + backbone -------------------------
    def backbone(self, rgb):
        """(B, 3, H, W) float32 -> context (B, 32m)."""
        import torch.nn.functional as F

        if rgb.dim() != 4 or rgb.shape[1] != 3:
            raise DimensionMismatch(f"rgb must be (B, 3, H, W), got {tuple(rgb.shape)}")
        t = self.t
        with _fp32_math():
            # half-pixel-centred bilinear with edge clamping == align_corners=False
            x = F.interpolate(rgb, size=(256, 256), mode="bilinear", align_corners=False)
            for i in range(1, 6):
                x = F.conv2d(x, t[f"backbone.conv{i}.weight"], t[f"backbone.conv{i}.bias"],
                             stride=2, padding=1)
                x = F.leaky_relu(x, _LEAKY_SLOPE)
                if i <= 4:
                    mean = x.mean(dim=(2, 3), keepdim=True)
                    var = x.var(dim=(2, 3), keepdim=True, unbiased=False)
                    inv = 1.0 / (var + _IN_EPS).sqrt()
                    x = ((x - mean) * inv * t[f"backbone.in{i}.scale"][None, :, None, None]
                         + t[f"backbone.in{i}.shift"][None, :, None, None])
            b, c, h, w = x.shape
            pooled = x.reshape(b, c, h // 4, 4, w // 4, 4).mean(dim=(3, 5))
            return pooled.reshape(b, -1).contiguous()

    # ---- reference network.py:131-169: the four heads ----------------------------
    def _head(self, name, ctx):
        t = self.t
        h = ctx @ t[f"{name}.fc1.weight"].T + t[f"{name}.fc1.bias"]
        return h @ t[f"{name}.fc2.weight"].T + t[f"{name}.fc2.bias"]

    def heads(self, ctx):
        """Context (B, 32m) -> dict of device tensors in the apply path's layout:
        u (B,3,3,d_t,n_s), s (B,3,3,n_s), vt (B,3,3,n_s,d_t), lw (B,3,3), lb (B,3),
        grid_planes (B,K,3,d_s,d_s), gw (B,K,3), gb (B,K)."""
        hp = self.hyper
        b = ctx.shape[0]
        d, n = hp.d_t, hp.n_s
        with _fp32_math():
            gp = self._head("grid_gen", ctx).reshape(b, hp.k, 3, hp.d_s, hp.d_s)
            gwb = self._head("gridw_gen", ctx).reshape(b, hp.k, 4)
            flat = self._head("lut_gen", ctx).reshape(b, 3, 3, 2 * d * n + n)
            lwb = self._head("lutw_gen", ctx).reshape(b, 3, 4)
        return {
            "u": flat[..., : d * n].reshape(b, 3, 3, d, n).contiguous(),
            "s": flat[..., d * n: d * n + n].contiguous(),
            "vt": flat[..., d * n + n:].reshape(b, 3, 3, d, n).transpose(-1, -2).contiguous(),
            "lw": lwb[..., :3].contiguous(),
            "lb": lwb[..., 3].contiguous(),
            "grid_planes": gp.contiguous(),
            "gw": gwb[..., :3].contiguous(),
            "gb": gwb[..., 3].contiguous(),
        }

    # ---- the whole pipeline on device ---------------------------------------------
    def tables(self, rgb):
        """Packed apply tables for a batch (backbone + heads + pack from factors)."""
        from . import device

        p = self.heads(self.backbone(rgb))
        return device.pack_tables_factors(p["u"], p["s"], p["vt"], p["lw"], p["lb"],
                                          p["grid_planes"], p["gw"], p["gb"])

    def enhance(self, rgb, out=None, nonfinite=None):
        """(B, 3, H, W) CUDA float32 -> enhanced image, all on device
        (``nonfinite``: optional int32 flag OR-ed with 1 on a NaN/Inf output)."""
        from . import device

        return device.apply(rgb, self.tables(rgb), out=out, nonfinite=nonfinite)

    def graphed(self, shape):
        """Enhance for a fixed (B, 3, H, W) as one CUDA-graph replay.

        At batch 1 the pipeline is ~40 small launches (resize, five convs with
        their norms, four heads, table packing, apply) and launch latency is
        most of its time; the graph replays them back to back.  Returns
        ``run(rgb) -> out``: ``rgb`` is copied into the graph's static input
        and ``out`` is the graph's static output tensor (overwritten by the
        next call).
        """
        import torch

        shape = tuple(int(v) for v in shape)
        x = torch.zeros(shape, dtype=torch.float32, device=self.device)
        out = torch.empty_like(x)
        flag = torch.zeros(1, dtype=torch.int32, device=self.device)  # NaN/Inf in the output
        with torch.cuda.device(self.device):  # capture on the generator's device
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):
                for _ in range(2):  # allocations, kernel attributes, texture objects
                    self.enhance(x, out=out, nonfinite=flag)
            torch.cuda.current_stream(self.device).wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            # relaxed: the apply may create a texture object over the graph pool's
            # table buffer while capturing (not a stream operation)
            with torch.cuda.graph(graph, capture_error_mode="relaxed"):
                flag.zero_()
                self.enhance(x, out=out, nonfinite=flag)

        def run(rgb):
            if tuple(rgb.shape) != shape:
                raise DimensionMismatch(f"graph was captured for {shape}, got {tuple(rgb.shape)}")
            x.copy_(rgb, non_blocking=True)
            graph.replay()
            return out

        run.graph = graph  # keeps the capture (and its memory pool) alive with the closure
        run.nonfinite = flag  # set by each replay
        return run

    def enhance_replayed(self, rgb, with_flag=False):
        """``enhance`` through a CUDA graph captured on the first call for
        each input shape (kept for the last four shapes).  The returned tensor
        is the graph's static output: consume it before the next call.
        ``with_flag``: also return the replay's int32 NaN/Inf output flag."""
        key = tuple(rgb.shape)
        cache = self.__dict__.setdefault("_graphs", {})
        if key not in cache:
            if len(cache) >= 4:
                cache.pop(next(iter(cache)))
            cache[key] = self.graphed(key)
        run = cache[key]
        out = run(rgb)
        return (out, run.nonfinite) if with_flag else out


def backbone_forward(img, params, device="cuda"):
    """Context vector (32m,) of one reference-style Image (network.py:115-128)."""
    import torch

    gen = params if isinstance(params, Generator) else Generator(params, device)
    rgb = torch.from_numpy(np.array(img.data, np.float32))[None].to(gen.device)
    return gen.backbone(rgb)[0].cpu().numpy()


def heads_forward(ctx, params, device="cuda"):
    """Host arrays (u, s, vt, lw, lb, grid_planes, gw, gb) from a context vector."""
    import torch

    gen = params if isinstance(params, Generator) else Generator(params, device)
    c = torch.from_numpy(np.ascontiguousarray(ctx, np.float32))[None].to(gen.device)
    return {k: v[0].cpu().numpy() for k, v in gen.heads(c).items()}


def run_model(img, params, fused=True, threads=1, device="cuda"):
    """Reference-facing ``network.run_model`` (network.py:179-186) on the GPU:
    Image in (host), enhanced Image out.  ``fused=False`` is accepted for
    signature compatibility and runs the same fused kernel (the naive
    multi-pass twin is an oracle, not a product path); ``threads`` is ignored."""
    import torch

    del fused, threads
    from . import transform

    reuse = isinstance(params, Generator)
    gen = params if reuse else Generator(params, device)
    if not reuse:  # a one-off call runs eagerly
        rgb = torch.from_numpy(np.array(img.data, np.float32))[None].to(gen.device)
        y = gen.enhance(rgb)[0].cpu().numpy()
        return transform._image_type(img)(img.width, img.height, y)
    # A Generator reused across calls replays a per-shape CUDA graph (batch 1
    # is launch-bound): one host copy into a page-locked input it keeps per
    # shape, H2D, replay, D2H straight into a fresh page-locked output that
    # the returned Image owns (no copy out), plus the replay's NaN/Inf flag,
    # so the host finiteness scan of the Image constructor is skipped when
    # the device found none (as fused_enhance does).
    shape = (1, 3, img.height, img.width)
    st = gen.__dict__.setdefault("_host_staging", {})
    if shape not in st:
        if len(st) >= 4:
            st.pop(next(iter(st)))
        st[shape] = (torch.empty(shape, dtype=torch.float32, pin_memory=True),
                     torch.zeros(1, dtype=torch.int32, pin_memory=True))
    pin_in, pin_flag = st[shape]
    pin_in[0].copy_(torch.from_numpy(np.asarray(img.data, np.float32)))
    pin_out = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    with torch.cuda.device(gen.device):
        y, flag = gen.enhance_replayed(pin_in, with_flag=True)  # the graph copies the input in (H2D)
        pin_out.copy_(y, non_blocking=True)
        pin_flag.copy_(flag, non_blocking=True)
        torch.cuda.current_stream(gen.device).synchronize()
    cls = transform._image_type(img)
    data = pin_out.numpy()[0]
    if int(pin_flag[0]) == 0 and issubclass(cls, _Image):
        return cls._trusted(img.width, img.height, data)
    return cls(img.width, img.height, data)  # validates (NonFiniteValue on NaN/Inf)
