"""Shared fixtures: golden-vector loader, the seeded rng, and the parity
comparators.

The ``gpu`` marker tags tests that need a B200; everything else runs on CPU.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
TOL64 = 1e-12  # conftest.py:15 of the reference (float64)
TOL32 = 1e-5  # north_star float32 tolerance


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    """List of case dicts from tests/golden/<name>.npz."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    n = int(z["n_cases"])
    cases = [dict() for _ in range(n)]
    for key in z.files:
        if key == "n_cases":
            continue
        ci, field = key.split("__", 1)
        v = z[key]
        cases[int(ci[1:])][field] = v.item() if v.ndim == 0 else v
    return cases


def assert_csc_equal(got, want, tol=TOL64, exact_values=False):
    """Structure bit-exact (as int64), values |d| <= tol*max(1,|ref|)
    (reference conftest.py:58-69) or bit-exact when exact_values."""
    gv, gr, go = (np.asarray(x) for x in got)
    wv, wr, wo = (np.asarray(x) for x in want)
    assert np.array_equal(go.astype(np.int64), wo.astype(np.int64)), "col_offsets differ"
    assert np.array_equal(gr.astype(np.int64), wr.astype(np.int64)), "row indices differ"
    gv = gv.astype(np.float64)
    if exact_values:
        assert np.array_equal(gv.view(np.int64), wv.astype(np.float64).view(np.int64)), "values not bit-exact"
    else:
        assert np.all(np.abs(gv - wv) <= tol * np.maximum(1.0, np.abs(wv))), "values outside tolerance"


def assert_close(a, b, tol=TOL64):
    assert abs(a - b) <= tol * max(1.0, abs(b)), (a, b)


@pytest.fixture
def rng():
    return np.random.default_rng(20260809)
