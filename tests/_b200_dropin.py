"""pytest plugin (``-p _b200_dropin``): installs the B200 path into the
reference package ``svdlut`` before the reference's own test modules import
it, so ``from svdlut.transform import fused_enhance`` in those tests binds the
GPU drop-in (paper_2508_16121_b200/plugin.py).  Used by
tests/test_gpu_reference_suite.py; SVDLUT_B200_GENERATOR=1 also routes
network.run_model through the GPU generator.  The terminal summary reports
how often each patched entry point ran, so the caller can prove the drop-in
(not the reference's numba code) served the tests."""

import collections
import functools
import os
import sys

_HANDLE = None
_CALLS = collections.Counter()


def _counted(mod, name):
    fn = getattr(mod, name)

    @functools.wraps(fn)
    def wrapper(*a, **k):
        _CALLS[name] += 1
        return fn(*a, **k)

    setattr(mod, name, wrapper)


def pytest_configure(config):
    global _HANDLE
    root = os.environ["SVDLUT_B200_ROOT"]
    if root not in sys.path:
        sys.path.insert(0, root)
    import svdlut.network
    import svdlut.svd
    import svdlut.transform

    from paper_2508_16121_b200 import plugin

    _HANDLE = plugin.install(generator=os.environ.get("SVDLUT_B200_GENERATOR") == "1")
    for name in ("fused_enhance", "naive_enhance", "apply_lut3d"):
        _counted(svdlut.transform, name)
        if hasattr(svdlut.network, name):
            setattr(svdlut.network, name, getattr(svdlut.transform, name))
    _counted(svdlut.svd, "reconstruct_lut")
    if os.environ.get("SVDLUT_B200_GENERATOR") == "1":
        _counted(svdlut.network, "run_model")


def pytest_terminal_summary(terminalreporter):
    import svdlut.transform

    mod = svdlut.transform.fused_enhance.__wrapped__.__module__
    terminalreporter.write_line(f"[b200-dropin] fused_enhance from {mod}; calls " +
                                " ".join(f"{k}={v}" for k, v in sorted(_CALLS.items())))


def pytest_unconfigure(config):
    if _HANDLE is not None:
        _HANDLE.uninstall()
