"""Install the B200 path into the reference package ``svdlut`` (drop-in).

    import svdlut
    from paper_2508_16121_b200 import plugin
    handle = plugin.install()        # svdlut now runs its hot path on the GPU
    ...
    handle.uninstall()

Patched names (the reference's own call sites):
  svdlut.transform.fused_enhance   transform.py:308   (tests import it by name)
  svdlut.network.fused_enhance     network.py:42      (bound at import by run_model)
  svdlut.svd.reconstruct_lut       svd.py:210         (called via module attribute)
  svdlut.transform.naive_enhance   transform.py:196   (multi-stage twin, f64 stage kernels)
  svdlut.network.naive_enhance     network.py:42      (run_model(fused=False))
  svdlut.transform.apply_lut3d     transform.py:93    (3D-LUT baseline)
  svdlut.network.run_model         network.py:179     (only with generator=True: the
                                                      backbone and heads run on the
                                                      GPU too, network.py here)

The wrappers keep the reference signatures, allocate the output raster
through ``svdlut.transform._alloc_raster`` (so ``_raster_hook`` observes exactly
one (3, H, W) allocation, transform.py:50-58), return the reference's own
``Image`` / ``Lut2DSet`` types, and re-raise errors as the reference's
exception classes of the same name (errors.py:4-31).
"""

import functools
import importlib

from . import errors as _errors

__all__ = ["install", "Handle"]


class Handle:
    def __init__(self, saved):
        self._saved = saved

    def uninstall(self):
        for (mod, name), fn in self._saved.items():
            setattr(mod, name, fn)
        self._saved = {}


def _translate(ref_errors):
    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            try:
                return fn(*args, **kwargs)
            except _errors.SvdLutError as exc:
                cls = getattr(ref_errors, type(exc).__name__, ref_errors.SvdLutError)
                raise cls(str(exc)) from exc
        return wrapper
    return deco


def install(package="svdlut", exact=False, generator=False):
    """Patch the reference package in place; returns a Handle to undo it.

    generator=True also routes ``network.run_model`` through the GPU generator
    path (resize + backbone + heads in PyTorch on device, then pack + apply)."""
    ref = importlib.import_module(package)
    ref_transform = importlib.import_module(f"{package}.transform")
    ref_network = importlib.import_module(f"{package}.network")
    ref_svd = importlib.import_module(f"{package}.svd")
    ref_errors = importlib.import_module(f"{package}.errors")
    from . import svd as b200_svd
    from . import transform as b200_transform

    @_translate(ref_errors)
    def fused_enhance(img, luts, lut_weights, grids, grid_weights, threads=1):
        return b200_transform.fused_enhance(img, luts, lut_weights, grids, grid_weights,
                                            threads=threads, exact=exact,
                                            alloc=ref_transform._alloc_raster)

    @_translate(ref_errors)
    def naive_enhance(img, luts, lut_weights, grids, grid_weights):
        return b200_transform.naive_enhance(img, luts, lut_weights, grids, grid_weights,
                                            alloc=ref_transform._alloc_raster)

    @_translate(ref_errors)
    def apply_lut3d(img, lut):
        return b200_transform.apply_lut3d(img, lut, alloc=ref_transform._alloc_raster)

    @_translate(ref_errors)
    def reconstruct_lut(svdlut):
        return b200_svd.reconstruct_lut(svdlut)

    from . import network as b200_network

    @_translate(ref_errors)
    def run_model(img, params, fused=True, threads=1):
        return b200_network.run_model(img, params, fused=fused, threads=threads)

    patches = [(ref_transform, "fused_enhance", fused_enhance),
               (ref_network, "fused_enhance", fused_enhance),
               (ref_transform, "naive_enhance", naive_enhance),
               (ref_network, "naive_enhance", naive_enhance),
               (ref_transform, "apply_lut3d", apply_lut3d),
               (ref_svd, "reconstruct_lut", reconstruct_lut)]
    if generator:
        patches.append((ref_network, "run_model", run_model))
    saved = {}
    for mod, name, fn in patches:
        saved[(mod, name)] = getattr(mod, name)
        setattr(mod, name, fn)
    del ref
    return Handle(saved)
