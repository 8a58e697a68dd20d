"""The reference's OWN tests, run on the B200 through the drop-in.

tools/install_reference.sh installs the unmodified reference package into the
git-ignored baseline/_ref/ together with a copy of its test suite; gpurun
ships it to the GPU box.  Each reference test module below runs in a fresh
pytest process with the ``_b200_dropin`` plugin, which calls
``plugin.install()`` before the modules import ``svdlut`` — so
``fused_enhance`` / ``naive_enhance`` / ``apply_lut3d`` /
``reconstruct_lut`` (and with the generator flag ``run_model``) in those
tests are the sm_100a kernels.  Covers, among others,
test_acceptance.py:32-50 (100 random models, fused vs naive ≤ 1e-5),
test_transform.py:270-296 (bitwise independence of ``threads``) and
:301-319 (exactly one raster allocation through ``_raster_hook``).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "svdlut_tests")


def _run(module, generator=False, extra=()):
    if not os.path.isdir(TESTS):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, TESTS, os.path.join(ROOT, "tests"), ROOT]),
               SVDLUT_B200_ROOT=ROOT, SVDLUT_B200_GENERATOR="1" if generator else "0",
               NUMBA_CACHE_DIR=os.path.join("/tmp", f"numba_b200_{os.getpid()}"), PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-p", "_b200_dropin", "-p", "no:cacheprovider", "-q",
           "-rfE", os.path.join(TESTS, module), *extra]
    res = subprocess.run(cmd, cwd=TESTS, env=env, capture_output=True, text=True, timeout=1800)
    tail = (res.stdout + res.stderr)[-4000:]
    assert res.returncode == 0, tail
    summary = [ln for ln in res.stdout.splitlines() if ln.startswith("[b200-dropin]")]
    assert summary and "paper_2508_16121_b200" in summary[0], "drop-in not active:\n" + tail
    assert "fused_enhance=" in summary[0] or "run_model=" in summary[0] or "reconstruct_lut=" in summary[0], tail
    return res.stdout


def test_reference_transform_suite_through_dropin():
    _run("test_transform.py")


def test_reference_acceptance_criteria_through_dropin():
    out = _run("test_acceptance.py", extra=["-k", "criterion_02 or criterion_03 or criterion_07 or criterion_08"])
    assert "passed" in out


def test_reference_svd_and_network_suites_through_dropin():
    _run("test_svd.py")
    _run("test_network.py", generator=True)
