"""Large-input construction / transpose (csrc/largen.cuh) against the oracle.

The pipeline takes over above the single-launch kernel's envelope (~1.2M
elements) and wherever that kernel's bucket tables do not fit (more than
~4M output columns); `as_set_engine(1)` forces it on small inputs too, so its
one-pass and two-pass variants, the oversized-bucket path and the error
reporting are all exercised here.  Reference: csc.canonicalize
(csc.py:148-193) and _kernels.transpose (_kernels.py:130-150); structure and
values bit-exact.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_1805_03380_b200 import _kernels, _lib

pytestmark = pytest.mark.gpu


@pytest.fixture
def engine():
    L = _lib.lib()

    def set_(e):
        _lib.check(L.as_set_engine(e))

    yield set_
    _lib.check(L.as_set_engine(0))


def _dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def _check_build(n_rows, n_cols, rows, cols, vals, dup="sum", idx=torch.int32, vdt=torch.float64):
    p, r, v, bad = _kernels.coo_to_csc(n_rows, n_cols, _dev(rows, idx), _dev(cols, idx), _dev(vals, vdt), dup)
    assert bad is None
    want = oracle.canonicalize(n_rows, n_cols, rows, cols, vals.astype(np.float64), dup)
    assert np.array_equal(p.cpu().numpy().astype(np.int64), want[2])
    assert np.array_equal(r.cpu().numpy().astype(np.int64), want[1])
    got = v.cpu().numpy().astype(np.float64)
    if vdt == torch.float64:
        assert np.array_equal(got.view(np.int64), want[0].view(np.int64))
    else:  # float32 sums vs the float64 oracle of the float32 inputs
        assert np.all(np.abs(got - want[0]) <= 1e-5 * np.maximum(1.0, np.abs(want[0])))


def _with_dups(rng, n_rows, n_cols, n, frac=0.05):
    rows = rng.integers(0, n_rows, n)
    cols = rng.integers(0, n_cols, n)
    k = int(n * frac)
    src = rng.integers(0, n - k, k)
    rows[n - k:], cols[n - k:] = rows[src], cols[src]
    vals = rng.uniform(-1, 1, n)
    vals[rng.integers(0, n, n // 100)] = 0.0
    return rows, cols, vals


@pytest.mark.parametrize("dup", ["sum", "last"])
def test_two_pass_build_3m(dup):
    rng = np.random.default_rng(11)
    rows, cols, vals = _with_dups(rng, 1_000_000, 1_000_000, 3_000_000)
    _check_build(1_000_000, 1_000_000, rows, cols, vals, dup)


def test_build_int64_f32_3m():
    rng = np.random.default_rng(12)
    rows, cols, vals = _with_dups(rng, 200_000, 300_000, 2_500_000)
    _check_build(200_000, 300_000, rows, cols, vals, idx=torch.int64, vdt=torch.float32)


def test_build_beyond_old_column_limit():
    # 12M output columns: the general kernel's tables stop at 8,192,000
    rng = np.random.default_rng(13)
    rows, cols, vals = _with_dups(rng, 12_000_000, 12_000_000, 1_500_000)
    _check_build(12_000_000, 12_000_000, rows, cols, vals)


@pytest.mark.parametrize("n,n_cols", [(0, 2500), (1, 2500), (5000, 2500), (300_000, 2500), (100_000, 2_000_000)])
def test_forced_pipeline_small(engine, n, n_cols):
    # single-pass (<= 256 buckets) and two-pass (2,000 column buckets) variants on small inputs
    engine(1)
    rng = np.random.default_rng(14 + n)
    rows, cols, vals = _with_dups(rng, 3000, n_cols, n) if n > 1 else (
        np.zeros(n, np.int64), np.zeros(n, np.int64), np.ones(n))
    _check_build(3000, n_cols, rows, cols, vals)


def test_forced_pipeline_heavy_column(engine):
    # one column with 200k entries (50k distinct rows, long duplicate runs):
    # buckets far above a tile take the oversized path
    engine(1)
    rng = np.random.default_rng(15)
    n = 400_000
    rows = np.where(rng.random(n) < 0.5, rng.integers(0, 50_000, n), rng.integers(0, 100_000, n))
    cols = np.where(rng.random(n) < 0.5, 777, rng.integers(0, 5000, n))
    vals = rng.standard_normal(n)
    _check_build(100_000, 5000, rows, cols, vals)
    _check_build(100_000, 5000, rows, cols, vals, "last")


def test_forced_pipeline_bad_triplet(engine):
    engine(1)
    rng = np.random.default_rng(16)
    n = 50_000
    rows, cols, vals = _with_dups(rng, 4000, 4000, n)
    rows[31_337] = 4000
    cols[40_000] = -1
    p, r, v, bad = _kernels.coo_to_csc(4000, 4000, _dev(rows, torch.int64), _dev(cols, torch.int64),
                                       _dev(vals, torch.float64))
    assert bad == 31_337
    keep = np.ones(n, bool)
    keep[[31_337, 40_000]] = False
    want = oracle.canonicalize(4000, 4000, rows[keep], cols[keep], vals[keep])
    assert np.array_equal(p.cpu().numpy(), want[2]) and np.array_equal(v.cpu().numpy(), want[0])


@pytest.mark.parametrize("vdt", [torch.float64, torch.float32])
def test_transpose_3m(vdt):
    rng = np.random.default_rng(17)
    n_rows, n_cols = 700_000, 900_000
    A = oracle.canonicalize(n_rows, n_cols, rng.integers(0, n_rows, 3_000_000), rng.integers(0, n_cols, 3_000_000),
                            rng.uniform(-1, 1, 3_000_000))
    vals = A[0].astype(np.float32) if vdt == torch.float32 else A[0]
    tp, tr, tv = _kernels.transpose(n_rows, n_cols, _dev(A[2], torch.int32), _dev(A[1], torch.int32), _dev(vals, vdt))
    want = oracle.transpose(n_rows, n_cols, vals.astype(np.float64), A[1], A[2])
    assert np.array_equal(tp.cpu().numpy().astype(np.int64), want[2])
    assert np.array_equal(tr.cpu().numpy().astype(np.int64), want[1])
    assert np.array_equal(tv.cpu().numpy().astype(np.float64), want[0])


def test_forced_transpose_sparse_columns(engine):
    # columns far sparser than a tile (uncached column pointers) and a heavy row
    engine(1)
    rng = np.random.default_rng(18)
    n_rows, n_cols, n = 5000, 3_000_000, 200_000
    rows = np.where(rng.random(n) < 0.2, 42, rng.integers(0, n_rows, n))
    A = oracle.canonicalize(n_rows, n_cols, rows, rng.integers(0, n_cols, n), rng.uniform(-1, 1, n))
    tp, tr, tv = _kernels.transpose(n_rows, n_cols, _dev(A[2], torch.int32), _dev(A[1], torch.int32),
                                    _dev(A[0], torch.float64))
    want = oracle.transpose(n_rows, n_cols, *A)
    assert np.array_equal(tp.cpu().numpy().astype(np.int64), want[2])
    assert np.array_equal(tr.cpu().numpy().astype(np.int64), want[1])
    assert np.array_equal(tv.cpu().numpy(), want[0])


def test_large_transpose_involution_10m():
    # size-independent property at BASELINE cfg 3 size: (A^T)^T == A, row counts
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    n = 1_000_000
    rows = torch.randint(0, n, (10_000_000,), device="cuda", dtype=torch.int32, generator=g)
    cols = torch.randint(0, n, (10_000_000,), device="cuda", dtype=torch.int32, generator=g)
    vals = torch.randn(10_000_000, device="cuda", dtype=torch.float32, generator=g)
    p, r, v, _ = _kernels.coo_to_csc(n, n, rows, cols, vals)
    tp, tr, tv = _kernels.transpose(n, n, p, r, v)
    pp, rr, vv = _kernels.transpose(n, n, tp, tr, tv)
    assert torch.equal(pp, p) and torch.equal(rr, r) and torch.equal(vv, v)
    assert torch.equal((tp[1:] - tp[:-1]).long(), torch.bincount(r.long(), minlength=n))


def test_flush_beyond_single_launch_envelope():
    # base CSC (1M nnz) ++ 1.5M element writes (overwrites of base entries, of
    # earlier writes, and 0.0 erasures): more elements than the single-launch
    # kernel takes, so the general bucket kernel runs (rbt.to_csc semantics)
    rng = np.random.default_rng(19)
    n_rows, n_cols = 400_000, 300_000
    base = oracle.canonicalize(n_rows, n_cols, rng.integers(0, n_rows, 1_000_000), rng.integers(0, n_cols, 1_000_000),
                               rng.uniform(-1, 1, 1_000_000))
    nl = 1_500_000
    lr = rng.integers(0, n_rows, nl)
    lc = rng.integers(0, n_cols, nl)
    bc = np.repeat(np.arange(n_cols), np.diff(base[2]))
    pick = rng.integers(0, base[1].shape[0], nl // 10)  # overwrite existing entries
    lr[: nl // 10], lc[: nl // 10] = base[1][pick], bc[pick]
    lr[-nl // 20:], lc[-nl // 20:] = lr[: nl // 20], lc[: nl // 20]  # rewrite earlier writes
    lv = rng.uniform(-1, 1, nl)
    lv[rng.integers(0, nl, nl // 50)] = 0.0  # erasures
    b = (_dev(base[2], torch.int32), _dev(base[1], torch.int32), _dev(base[0], torch.float64))
    p, r, v, bad = _kernels.flush_log(n_rows, n_cols, b, _dev(lr, torch.int32), _dev(lc, torch.int32),
                                      _dev(lv, torch.float64))
    assert bad is None
    want = oracle.flush(n_rows, n_cols, base, lr, lc, lv)
    assert np.array_equal(p.cpu().numpy().astype(np.int64), want[2])
    assert np.array_equal(r.cpu().numpy().astype(np.int64), want[1])
    assert np.array_equal(v.cpu().numpy(), want[0])


@pytest.mark.parametrize("dup", ["sum", "last"])
def test_general_bucket_kernel_engine(engine, dup):
    # engine 2: the general bucket kernel (persist.cuh) for construction and transpose
    engine(2)
    rng = np.random.default_rng(20)
    rows, cols, vals = _with_dups(rng, 50_000, 40_000, 600_000)
    _check_build(50_000, 40_000, rows, cols, vals, dup)
    A = oracle.canonicalize(50_000, 40_000, rows, cols, vals)
    tp, tr, tv = _kernels.transpose(50_000, 40_000, _dev(A[2], torch.int32), _dev(A[1], torch.int32),
                                    _dev(A[0], torch.float64))
    want = oracle.transpose(50_000, 40_000, *A)
    assert np.array_equal(tp.cpu().numpy().astype(np.int64), want[2]) and np.array_equal(tv.cpu().numpy(), want[0])
