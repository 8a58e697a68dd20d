"""pytest plugin (``-p _b200_dropin``): installs the B200 path into the
reference package ``svdlut`` before the reference's own test modules import
it, so ``from svdlut.transform import fused_enhance`` in those tests binds the
GPU drop-in (paper_2508_16121_b200/plugin.py).  Used by
tests/test_gpu_reference_suite.py; SVDLUT_B200_GENERATOR=1 also routes
network.run_model through the GPU generator."""

import os
import sys

_HANDLE = None


def pytest_configure(config):
    global _HANDLE
    root = os.environ["SVDLUT_B200_ROOT"]
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_2508_16121_b200 import plugin

    _HANDLE = plugin.install(generator=os.environ.get("SVDLUT_B200_GENERATOR") == "1")
    config.addinivalue_line("markers", "b200_dropin: reference tests run through the B200 drop-in")


def pytest_report_header(config):
    import svdlut.transform

    return f"svdlut.transform.fused_enhance -> {svdlut.transform.fused_enhance.__module__}"


def pytest_unconfigure(config):
    if _HANDLE is not None:
        _HANDLE.uninstall()
