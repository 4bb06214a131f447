"""The reference package itself, routed through this back end.

`ref_kernels.install(autosparse)` swaps the reference's flat-array kernel
module (ops._kernels, expr._kernels; _kernels.py:1-175), csc.canonicalize
(csc.py:148-193) and the element-write store with rbt.to_csc / rbt.from_csc
(rbt.py:303-476) for the GPU path.  Each scenario below runs the reference's
own public API (SpMat constructors, element writes, +, -, @, .t(), scalar *,
SpMV, the expression engine with its fused-trace rewrite, reductions and the
construction-funnelled ops) twice on the same seeded inputs: once on the
stock reference (numpy / numba on the host) and once swapped; the results
must be identical (trace: 1e-12 relative).

The reference is the pip-installed copy under baseline/_ref (bench.py's
reference arm ships it to the GPU box); without it these tests skip.
"""

import os
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "autosparse")):
        pytest.skip("reference package not installed under baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "as_numba_cache"))
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import autosparse

    return autosparse


def _triplets(rng, n_r, n_c, n, dup_frac=0.1):
    rows = rng.integers(0, n_r, n)
    cols = rng.integers(0, n_c, n)
    k = int(n * dup_frac)
    rows[-k:], cols[-k:] = rows[:k], cols[:k]  # duplicates to be summed
    vals = rng.uniform(-1, 1, n)
    vals[: max(1, n // 50)] = 0.0  # explicit zeros: pruned unless a duplicate revives them
    return [(int(r), int(c), float(v)) for r, c, v in zip(rows, cols, vals)]


def _arrays(m):
    d = m.csc()
    return np.asarray(d.values), np.asarray(d.row_indices), np.asarray(d.col_offsets)


def scenario(pkg, seed):
    """Reference API calls only; returns every observable result."""
    SpMat, ops = pkg.SpMat, pkg.ops
    rng = np.random.default_rng(seed)
    out = {}
    n_r, n_c, n = 120, 90, 4000
    A = SpMat.from_triplets(n_r, n_c, _triplets(rng, n_r, n_c, n))
    B = SpMat.from_triplets(n_r, n_c, _triplets(rng, n_r, n_c, n))
    C = SpMat.from_triplets(n_c, 70, _triplets(rng, n_c, 70, 3000))
    out["A"] = _arrays(A)
    out["B"] = _arrays(B)
    out["A_last"] = _arrays(SpMat.from_triplets(n_r, n_c, _triplets(rng, n_r, n_c, 2000), dup="last"))
    out["A+B"] = _arrays(A + B)
    out["A-B"] = _arrays(A - B)
    out["A-A"] = _arrays(A - A)
    out["scaled_sum"] = _arrays(ops.scaled_sum(A, B, -0.75))
    out["2.5*A"] = _arrays(A * 2.5)
    out["A.t()"] = _arrays(A.t())
    out["A@C"] = _arrays(A @ C)
    out["At@B"] = _arrays(ops.matmul(A.t(), B))
    x = rng.uniform(-1, 1, n_c)
    x[::7] = 0.0
    out["A@x"] = (A @ x,)
    v = rng.uniform(-1, 1, n_r)
    out["v@A"] = (v @ A,)
    # element writes: fresh matrix, overwrites, erase by 0.0, accumulate
    W = SpMat.zeros(300, 200)
    wr = rng.integers(0, 300, 3000)
    wc = rng.integers(0, 200, 3000)
    wv = rng.uniform(-1, 1, 3000)
    for i in range(3000):
        W[int(wr[i]), int(wc[i])] = float(wv[i])
    for i in range(0, 3000, 9):  # erase some
        W[int(wr[i]), int(wc[i])] = 0.0
    for i in range(0, 3000, 13):
        W.accumulate(int(wr[i]), int(wc[i]), 0.5)
    out["W"] = _arrays(W)
    out["W.get"] = (np.array([W[int(wr[i]), int(wc[i])] for i in range(0, 3000, 11)]),)
    # writes on a CSC-resident matrix: in-place patch, then a structural write
    A2 = A.copy()
    d = A2.csc()
    r0 = int(d.row_indices[0])
    A2[r0, 0] = 3.25
    A2[n_r - 1, n_c - 1] = 1.5
    A2[r0, 0] = 0.0
    out["A2"] = _arrays(A2)
    out["conv"] = (np.array(sorted(str(k) for k in A2.conversions.items())),)
    # expression engine: fused trace (P1), scaled sum (P4), transposed operand
    E = pkg.lift
    out["trace"] = pkg.evaluate(pkg.Trace(E(A).t() @ E(B)))
    out["expr_ss"] = _arrays(pkg.evaluate(E(A) + E(B) * 0.5))
    out["expr_mix"] = _arrays(pkg.evaluate((E(A) + E(B)) * 0.5 @ E(C)))
    # reductions / funnelled ops (§8f-2)
    out["sum0"] = (ops.sum_dim(A, 0),)
    out["max1"] = (ops.max_dim(A, 1),)
    out["kron"] = _arrays(ops.kron(SpMat.from_triplets(3, 2, [(0, 0, 1.0), (2, 1, -2.0)]), C))
    out["repmat"] = _arrays(ops.repmat(C, 2, 3))
    out["speye"] = _arrays(ops.speye(40, 30))
    out["sprandu"] = _arrays(ops.sprandu(200, 150, 0.05, seed=seed))
    out["from_dense"] = _arrays(SpMat.from_dense(A.to_dense()))
    return out


def _same(a, b):
    return a.shape == b.shape and (a.dtype.kind == "U" and np.array_equal(a, b)
                                   or np.array_equal(np.asarray(a, np.float64).view(np.int64),
                                                     np.asarray(b, np.float64).view(np.int64)))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_reference_api_through_gpu_backend(ref, seed):
    from paper_1805_03380_b200 import ref_kernels

    want = scenario(ref, seed)
    undo = ref_kernels.install(ref)
    try:
        got = scenario(ref, seed)
    finally:
        undo()
    assert set(got) == set(want)
    for k in want:
        if k == "trace":
            assert abs(got[k] - want[k]) <= 1e-12 * max(1.0, abs(want[k])), (got[k], want[k])
            continue
        for g, w in zip(got[k], want[k]):
            assert _same(np.asarray(g), np.asarray(w)), k


def test_install_routes_through_gpu(ref):
    """The swapped calls really reach the device kernels (no host path)."""
    from paper_1805_03380_b200 import _kernels, ref_kernels

    calls = []
    orig = _kernels.coo_to_csc, _kernels.flush_log

    def spy(name, fn):
        def f(*a, **k):
            calls.append(name)
            return fn(*a, **k)
        return f

    _kernels.coo_to_csc, _kernels.flush_log = spy("build", orig[0]), spy("flush", orig[1])
    undo = ref_kernels.install(ref)
    try:
        M = ref.SpMat.from_triplets(5, 4, [(0, 0, 1.0), (4, 3, 2.0), (0, 0, 1.0)])
        M[1, 1] = 5.0
        d = M.csc()
        assert isinstance(d, ref.CscData)
        assert d.values.tolist() == [2.0, 5.0, 2.0]
    finally:
        undo()
        _kernels.coo_to_csc, _kernels.flush_log = orig
    assert "build" in calls and "flush" in calls


def test_install_errors_match(ref):
    from paper_1805_03380_b200 import ref_kernels

    undo = ref_kernels.install(ref)
    try:
        with pytest.raises(ref.CoordinateError):
            ref.SpMat.from_triplets(3, 3, [(0, 0, 1.0), (3, 0, 1.0)])
        with pytest.raises(ValueError):
            ref.csc.canonicalize(ref.Dims(2, 2), np.array([0]), np.array([0]), np.array([1.0]), "max")
        with pytest.raises(ref.ShapeError):
            ref.SpMat.zeros(2, 3) + ref.SpMat.zeros(3, 2)
    finally:
        undo()
