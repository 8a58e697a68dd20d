"""Shared test setup.

* ``gpu`` marker: tests that need a B200 (run with ``-m gpu`` on the GPU box).
* The CPU oracle (``oracle/``) is test infrastructure; it is built on demand.
* Golden vectors come from the real reference (tests/golden/make_golden.py).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build()
    return oracle


def golden_case(g, name):
    keys = ("rgb", "lp", "lw", "lb", "gp", "gw", "gb", "want")
    return {k: g[f"tr_{name}_{k}"] for k in keys}


# conftest-style generators (reference tests/conftest.py:14-45 distributions)
def make_inputs(w, h, d_t=9, d_s=5, k=6, seed=0, low=0.0, high=1.0):
    rng = np.random.default_rng(seed)
    rgb = rng.uniform(low, high, (3, h, w)).astype(np.float32)
    lp = rng.random((3, 3, d_t, d_t)).astype(np.float32)
    lw = rng.uniform(-1, 1, (3, 3)).astype(np.float32)
    lb = rng.uniform(-0.5, 0.5, 3).astype(np.float32)
    gp = rng.uniform(-1, 1, (k, 3, d_s, d_s)).astype(np.float32)
    gw = rng.uniform(-1, 1, (k, 3)).astype(np.float32)
    gb = rng.uniform(-0.5, 0.5, k).astype(np.float32)
    return dict(rgb=rgb, lp=lp, lw=lw, lb=lb, gp=gp, gw=gw, gb=gb)
