"""Edge cases and the rarely taken kernel paths, against the oracle:
empty operands, degenerate shapes, a bucket far above the shared-memory tile
(global row-prefix split), a single run of thousands of duplicates (global
radix fallback), Zipf-skewed SpGEMM columns with heavy row collisions
(pre-bucketed oversized path), trace columns above the register and shared
buffers (global search path), SpMM chunk remainders and empty rows."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_close, assert_csc_equal

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _t(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def _csc(c):
    v, r, p = c
    return _t(p, torch.int32), _t(r, torch.int32), _t(v, torch.float64)


def _np(csc):
    p, r, v = csc[:3]
    return v.cpu().numpy(), r.cpu().numpy(), p.cpu().numpy()


@pytest.fixture(scope="module")
def K():
    from paper_1805_03380_b200 import _kernels

    return _kernels


def _build(K, n_rows, n_cols, rows, cols, vals, dup="sum"):
    p, r, v, bad = K.coo_to_csc(n_rows, n_cols, _t(rows, torch.int64), _t(cols, torch.int64),
                                _t(vals, torch.float64), dup)
    assert bad is None
    return (v.cpu().numpy(), r.cpu().numpy(), p.cpu().numpy())


@pytest.mark.parametrize("shape", [(0, 0), (5, 0), (0, 5), (1, 1), (7, 3)])
def test_build_empty(K, shape):
    n_rows, n_cols = shape
    got = _build(K, n_rows, n_cols, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    assert_csc_equal(got, oracle.canonicalize(n_rows, n_cols, [], [], []), exact_values=True)


@pytest.mark.parametrize("dup", ["sum", "last"])
def test_build_one_huge_duplicate_run(K, rng, dup):
    # 6000 copies of one key (the radix fallback of a single bin above the
    # tile) next to a light background; pairwise order must match numpy
    n = 6000
    rows = np.concatenate([np.full(n, 3), rng.integers(0, 50, 2000)])
    cols = np.concatenate([np.full(n, 7), rng.integers(0, 40, 2000)])
    vals = rng.uniform(-1, 1, rows.shape[0])
    perm = rng.permutation(rows.shape[0])
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    got = _build(K, 50, 40, rows, cols, vals, dup)
    assert_csc_equal(got, oracle.canonicalize(50, 40, rows, cols, vals, dup), exact_values=True)


def test_build_single_heavy_column(K, rng):
    # 50k elements in one column over 200k rows: a bucket 25x the tile,
    # split into row-prefix bins in global memory
    n = 50_000
    rows = rng.integers(0, 200_000, n)
    cols = np.where(rng.random(n) < 0.9, 5, rng.integers(0, 64, n))
    vals = rng.uniform(-1, 1, n)
    got = _build(K, 200_000, 64, rows, cols, vals)
    assert_csc_equal(got, oracle.canonicalize(200_000, 64, rows, cols, vals), exact_values=True)


def test_build_many_columns_few_entries(K, rng):
    n_cols, n = 3_000_000, 20_000
    rows, cols, vals = rng.integers(0, 1000, n), rng.integers(0, n_cols, n), rng.uniform(-1, 1, n)
    got = _build(K, 1000, n_cols, rows, cols, vals)
    assert_csc_equal(got, oracle.canonicalize(1000, n_cols, rows, cols, vals), exact_values=True)


def test_build_all_cancel(K):
    rows = np.array([0, 1, 0, 1])
    cols = np.array([0, 0, 0, 0])
    vals = np.array([1.5, -2.0, -1.5, 2.0])
    got = _build(K, 2, 1, rows, cols, vals)
    assert got[0].shape[0] == 0 and got[2].tolist() == [0, 0]


def test_flush_erase_everything_and_empty_log(K, rng):
    base = oracle.canonicalize(30, 20, rng.integers(0, 30, 200), rng.integers(0, 20, 200), rng.uniform(-1, 1, 200))
    v, r, p = base
    cols = np.repeat(np.arange(20), np.diff(p))
    dbase = _csc(base)
    # erase every entry
    got = K.flush_log(30, 20, dbase, _t(r, torch.int32), _t(cols, torch.int32), _t(np.zeros(r.shape[0]), torch.float64))
    assert int(got[1].shape[0]) == 0
    # empty log: the base comes back unchanged
    e = torch.zeros(0, dtype=torch.int32, device=DEV)
    got = K.flush_log(30, 20, dbase, e, e, torch.zeros(0, dtype=torch.float64, device=DEV))
    assert_csc_equal(_np(got), base, exact_values=True)


def test_transpose_degenerate(K, rng):
    for n_rows, n_cols, n in [(1, 500, 300), (500, 1, 300), (3, 3, 0)]:
        a = oracle.canonicalize(n_rows, n_cols, rng.integers(0, n_rows, n), rng.integers(0, n_cols, n),
                                rng.uniform(-1, 1, n))
        got = K.transpose(n_rows, n_cols, *_csc(a))
        assert_csc_equal(_np(got), oracle.transpose(n_rows, n_cols, *a), exact_values=True)


def test_add_with_empty_and_cancelling(K, rng):
    a = oracle.canonicalize(40, 30, rng.integers(0, 40, 300), rng.integers(0, 30, 300), rng.uniform(-1, 1, 300))
    empty = oracle.canonicalize(40, 30, [], [], [])
    for x, y, al, be in [(a, empty, 1.0, 1.0), (empty, a, 2.0, -1.0), (empty, empty, 1.0, 1.0), (a, a, 1.0, -1.0),
                         (a, a, 0.0, 3.0)]:
        got = K.linear_combine(40, 30, _csc(x), _csc(y), al, be)
        assert_csc_equal(_np(got), oracle.linear_combine(30, *x, *y, al, be), exact_values=True)


def test_add_tile_boundaries(K):
    # the merge is cut into fixed tiles of merged positions: coincident pairs
    # straddle tile edges, tiles span thousands of empty columns, one column
    # spans many tiles, everything cancels
    rng = np.random.default_rng(31)
    a = oracle.canonicalize(2000, 2000, rng.integers(0, 2000, 300000), rng.integers(0, 2000, 300000),
                            rng.uniform(-1, 1, 300000))
    keep = rng.random(a[0].shape[0]) < 0.5
    half = oracle.canonicalize(2000, 2000, a[1][keep], np.repeat(np.arange(2000), np.diff(a[2]))[keep],
                               a[0][keep] * 3.0)
    sparse_cols = oracle.canonicalize(50, 2000000, rng.integers(0, 50, 9000), rng.integers(0, 2000000, 9000),
                                      rng.uniform(-1, 1, 9000))
    sparse_cols2 = oracle.canonicalize(50, 2000000, rng.integers(0, 50, 7000), rng.integers(0, 2000000, 7000),
                                       rng.uniform(-1, 1, 7000))
    one_col = oracle.canonicalize(1000000, 1, rng.integers(0, 1000000, 300000), np.zeros(300000, np.int64),
                                  rng.uniform(-1, 1, 300000))
    one_col2 = oracle.canonicalize(1000000, 1, rng.integers(0, 1000000, 200000), np.zeros(200000, np.int64),
                                   rng.uniform(-1, 1, 200000))
    cases = [(2000, 2000, a, a, 1.0, 1.0), (2000, 2000, a, a, 1.0, -1.0), (2000, 2000, a, half, 1.0, 1.0),
             (2000, 2000, half, a, -0.5, 2.0), (50, 2000000, sparse_cols, sparse_cols2, 1.0, 1.0),
             (1000000, 1, one_col, one_col2, 1.0, 1.0), (1000000, 1, one_col, one_col, 2.0, -2.0),
             (2000, 2000, a, half, 0.0, 1.0), (2000, 2000, half, a, 1.0, 0.0), (2000, 2000, a, half, 1e-300, 1e-300)]
    for n_rows, n_cols, x, y, al, be in cases:
        got = K.linear_combine(n_rows, n_cols, _csc(x), _csc(y), al, be)
        assert_csc_equal(_np(got), oracle.linear_combine(n_cols, *x, *y, al, be), exact_values=True)


def test_spgemm_empty_and_zero_products(K, rng):
    a = oracle.canonicalize(20, 10, rng.integers(0, 20, 50), rng.integers(0, 10, 50), rng.uniform(-1, 1, 50))
    empty_b = oracle.canonicalize(10, 15, [], [], [])
    got = K.spgemm(20, 10, 15, _csc(a), _csc(empty_b))
    assert int(got[1].shape[0]) == 0 and got[0].cpu().tolist() == [0] * 16
    # B only touches empty columns of A: zero products
    a2 = oracle.canonicalize(20, 10, rng.integers(0, 20, 50), rng.integers(0, 5, 50), rng.uniform(-1, 1, 50))
    b2 = oracle.canonicalize(10, 15, rng.integers(5, 10, 40), rng.integers(0, 15, 40), rng.uniform(-1, 1, 40))
    got = K.spgemm(20, 10, 15, _csc(a2), _csc(b2))
    assert_csc_equal(_np(got), oracle.spgemm(20, *a2, *b2, 15), exact_values=True)


def test_spgemm_heavy_column_row_collisions(K, rng):
    # one B column selecting 300 A columns that all hit the same few rows:
    # a pre-bucketed oversized bucket whose runs are hundreds long
    m, k, n = 64, 400, 20
    a_rows = rng.integers(0, 8, 4000)
    a_cols = rng.integers(0, k, 4000)
    a = oracle.canonicalize(m, k, a_rows, a_cols, rng.standard_normal(4000))
    b_rows = np.concatenate([rng.choice(k, 300, replace=False), rng.integers(0, k, 60)])
    b_cols = np.concatenate([np.full(300, 4), rng.integers(0, n, 60)])
    b = oracle.canonicalize(k, n, b_rows, b_cols, rng.standard_normal(b_rows.shape[0]))
    got = K.spgemm(m, k, n, _csc(a), _csc(b))
    assert_csc_equal(_np(got), oracle.spgemm(m, *a, *b, n), exact_values=True)


def test_trace_long_columns(K, rng):
    # columns of ~100 (register path), ~600 (shared buffer) and ~3000
    # entries (global search) in the same matrices
    n_rows = 20_000
    lens = np.array([100] * 50 + [600] * 8 + [3000] * 3)
    n_cols = lens.shape[0]

    def mk(seed):
        g = np.random.default_rng(seed)
        rows = np.concatenate([g.choice(n_rows, L, replace=False) for L in lens])
        cols = np.repeat(np.arange(n_cols), lens)
        return oracle.canonicalize(n_rows, n_cols, rows, cols, g.uniform(-1, 1, rows.shape[0]))

    a, b = mk(1), mk(2)
    got = K.fused_trace(n_rows, n_cols, _csc(a), _csc(b)).cpu().numpy()
    assert_close(float(got[0]), oracle.fused_trace(n_cols, *a, *b))


@pytest.mark.parametrize("k", [1, 3, 16, 17, 33])
def test_spmm_chunk_remainders_empty_rows(K, rng, k):
    n_rows, n_cols = 300, 200
    rows = rng.integers(0, n_rows // 2, 3000)  # upper half of the rows stays empty
    a = oracle.canonicalize(n_rows, n_cols, rows, rng.integers(0, n_cols, 3000), rng.standard_normal(3000))
    at = oracle.transpose(n_rows, n_cols, *a)
    csr = (_t(at[2], torch.int32), _t(at[1], torch.int32), _t(at[0], torch.float64))
    X = rng.standard_normal((n_cols, k))
    X[rng.random(X.shape) < 0.1] = 0.0
    got = K.spmm(n_rows, n_cols, csr, torch.as_tensor(np.asfortranarray(X), device=DEV)).cpu().numpy()
    want = oracle.spmm(*a, X, n_rows, n_cols)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("shape", [(200_000, 300_000, 3_000_000), (5_000, 2_000_000, 4_000_000),
                                   (60_000, 40_000, 2_000_000)])
def test_build_and_transpose_two_level_scatter(K, rng, shape):
    # element data beyond L2: the two-level (super-bucket) scatter path; the
    # 2e6 case: CTA chunks above the shared-memory staging, below the
    # two-level threshold (the direct per-element scatter)
    n_rows, n_cols, n = shape
    rows, cols = rng.integers(0, n_rows, n), rng.integers(0, n_cols, n)
    vals = rng.uniform(-1, 1, n)
    got = _build(K, n_rows, n_cols, rows, cols, vals)
    want = oracle.canonicalize(n_rows, n_cols, rows, cols, vals)
    assert_csc_equal(got, want, exact_values=True)
    t = K.transpose(n_rows, n_cols, *_csc(want))
    assert_csc_equal(_np(t), oracle.transpose(n_rows, n_cols, *want), exact_values=True)


@pytest.mark.parametrize("heavy", [1500, 2047, 2049, 20000])
def test_spgemm_dense_column_path_boundaries(K, rng, heavy):
    # light columns then one column of `heavy` products in the same
    # pre-bucketed bucket: the bucket is above the tile, its last column
    # takes the dense path -- with keys (<= 2048 products) or row-only
    # products (> 2048); collisions from two A columns hitting the same rows
    m = 30_000
    a_rows = [rng.choice(m, heavy, replace=False), rng.choice(m, heavy // 2, replace=False)]
    a_cols = [np.zeros(heavy, np.int64), np.ones(heavy // 2, np.int64)]
    a_rows.append(rng.integers(0, m, 2000))
    a_cols.append(rng.integers(2, 1000, 2000))
    ar, ac = np.concatenate(a_rows), np.concatenate(a_cols)
    a = oracle.canonicalize(m, 1000, ar, ac, rng.standard_normal(ar.shape[0]))
    n = 800
    b_rows = [rng.integers(2, 1000, 768), np.array([0, 1])]
    b_cols = [np.repeat(np.arange(384), 2), np.array([384, 384])]
    b_rows.append(rng.integers(0, 1000, 600))
    b_cols.append(rng.integers(385, n, 600))
    br, bc = np.concatenate(b_rows), np.concatenate(b_cols)
    bv = rng.standard_normal(br.shape[0])
    bv[-5:] = 0.0  # explicit zeros dropped by canonicalize
    b = oracle.canonicalize(1000, n, br, bc, bv)
    got = K.spgemm(m, 1000, n, _csc(a), _csc(b))
    assert_csc_equal(_np(got), oracle.spgemm(m, *a, *b, n), exact_values=True)


def test_spgemm_dense_column_cancellation_and_underflow(K):
    # exact cancellations and underflowing products inside a dense column are
    # pruned like the reference's `!= 0.0` filter
    m = 5000
    rows0 = np.arange(3000)
    a = oracle.canonicalize(m, 3, np.concatenate([rows0, rows0, rows0[:10]]),
                            np.concatenate([np.zeros(3000, np.int64), np.ones(3000, np.int64), np.full(10, 2)]),
                            np.concatenate([np.full(3000, 1.5), np.full(3000, -1.5), np.full(10, 1e-300)]))
    b = oracle.canonicalize(3, 2, np.array([0, 1, 2, 0]), np.array([0, 0, 0, 1]), np.array([2.0, 2.0, 1e-300, 1.0]))
    got = K.spgemm(m, 3, 2, _csc(a), _csc(b))
    want = oracle.spgemm(m, *a, *b, 2)
    assert_csc_equal(_np(got), want, exact_values=True)
    assert int(want[2][1]) == 0  # column 0 cancels / underflows to nothing


@pytest.mark.parametrize("n_rows,n_cols", [(1000, 1000), (400000, 30), (100000, 20)])
def test_add_persistent_tile_reuse(K, n_rows, n_cols):
    # ~2M merged positions -> ~1000 tiles of 2048, more than the resident grid
    # (4 CTAs x 148 SMs), so persistent CTAs take second tiles; the columns are
    # low (< 2048), where leftover per-tile shared state would read as column
    # marks (mark / excl shared storage)
    rng = np.random.default_rng(77)
    n = 1100000
    a = oracle.canonicalize(n_rows, n_cols, rng.integers(0, n_rows, n), rng.integers(0, n_cols, n),
                            rng.uniform(-1, 1, n))
    b = oracle.canonicalize(n_rows, n_cols, rng.integers(0, n_rows, n), rng.integers(0, n_cols, n),
                            rng.uniform(-1, 1, n))
    assert a[0].shape[0] + b[0].shape[0] > 2048 * 4 * 148
    for al, be in [(1.0, 1.0), (1.0, -1.0), (0.5, 2.0)]:
        got = K.linear_combine(n_rows, n_cols, _csc(a), _csc(b), al, be)
        assert_csc_equal(_np(got), oracle.linear_combine(n_cols, *a, *b, al, be), exact_values=True)
