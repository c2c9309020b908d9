"""Shared pytest configuration.

Markers: ``gpu`` — needs a B200 (the driver runs ``-m gpu`` on a GPU box, ``-m "not gpu"`` here).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    # tests/test_gpu_checked.py re-runs GPU test files in a subprocess against the CHECKED library
    # (make rg-checked: device bounds / invariant checks compiled in); test infrastructure only
    lib = os.environ.get("RG_TEST_CHECKED_LIB")
    if lib:
        from paper_1807_09467_b200 import rg as _rg
        _rg._lib = _rg.load(lib)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def pytest_sessionfinish(session, exitstatus):
    """Under RG_TEST_CHECKED_LIB: record which librg*.so files this process mapped (the checked-run
    test asserts it was the checked library)."""
    mark = os.environ.get("RG_TEST_CHECKED_MARK")
    if mark:
        try:
            maps = open("/proc/self/maps").read().splitlines()
        except OSError:
            maps = []
        libs = sorted({ln.split()[-1] for ln in maps if "librg" in ln})
        with open(mark, "w") as f:
            f.write("\n".join(libs) + "\n")

