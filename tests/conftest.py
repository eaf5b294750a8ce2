import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: larger parity cases (full-size configs)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_err(a, b, floor=1e-300):
    """Largest relative difference over finite entries; inf when the NaN
    positions differ (a bin that received 1/0 is NaN in the reference)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if not np.array_equal(np.isnan(a), np.isnan(b)):
        return float("inf")
    m = ~np.isnan(a)
    if not m.any():
        return 0.0
    a, b = a[m], b[m]
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def surfaces_close(a, b, rel_tol=1e-9, abs_tol=1e-12):
    """testutil::rel_close elementwise (proj/tests/helpers.hpp:141-152), with
    NaN required in the same places."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if not np.array_equal(np.isnan(a), np.isnan(b)):
        return False
    m = ~np.isnan(a)
    a, b = a[m], b[m]
    tol = np.maximum(abs_tol, rel_tol * np.maximum(np.abs(a), np.abs(b)))
    return bool(np.all(np.abs(a - b) <= tol))
