"""Column-merge SpMM straight over the CSC (as_spmm_csc_f32, the first product
on a fresh CSC handle) against the float64 oracle: one mat_times_vec per
dense column (_kernels.py:118-127), float32 tolerance 1e-5
relative (the north star's float32 bound; additions run in arrival order).
Covers the bulk-copy (TMA) staging path, the plain-load path (unaligned B),
chunk widths that are not a multiple of 16, heavy columns spanning many
tiles, hypersparse column ranges (B read from global memory), empty
matrices, and the SpMat dispatch (first product by columns, second through
the cached CSR)."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def K():
    from paper_1805_03380_b200 import _kernels

    return _kernels


def _case(rng, n_rows, n_cols, rows, cols):
    a = oracle.canonicalize(n_rows, n_cols, rows, cols, rng.standard_normal(rows.shape[0]))
    return (a[0].astype(np.float32).astype(np.float64), a[1], a[2])


def _dev(a):
    v, r, p = a
    return (torch.as_tensor(p, dtype=torch.int32, device=DEV), torch.as_tensor(r, dtype=torch.int32, device=DEV),
            torch.as_tensor(v, dtype=torch.float32, device=DEV))


def _check(C, want):
    C = C.cpu().numpy().astype(np.float64)
    assert C.shape == want.shape
    assert np.all(np.abs(C - want) <= 1e-5 * np.maximum(1.0, np.abs(want))), np.max(np.abs(C - want))


def _B(rng, n, k, ld=None, offset=0):
    """column-major float32 B (n x k) with leading dimension ld, starting
    `offset` floats into its storage (offset 1: not 16-byte aligned)"""
    ld = ld or n
    store = torch.zeros(offset + ld * k, dtype=torch.float32, device=DEV)
    Bn = rng.standard_normal((n, k)).astype(np.float32)
    Bn[rng.random((n, k)) < 0.05] = 0.0
    view = store[offset:].as_strided((n, k), (1, ld))
    view.copy_(torch.as_tensor(Bn, device=DEV))
    return view, Bn.astype(np.float64)


@pytest.mark.parametrize("k", [1, 5, 16, 17, 64])
@pytest.mark.parametrize("n_rows", [30000, 30003])  # (30003: C's columns unaligned, a partial row quad)
def test_spmm_csc_uniform(K, k, n_rows):
    rng = np.random.default_rng(50 + k)
    n_cols, nnz = 20000, 200000
    a = _case(rng, n_rows, n_cols, rng.integers(0, n_rows, nnz), rng.integers(0, n_cols, nnz))
    B, Bn = _B(rng, n_cols, k)
    want = oracle.spmm(*a, Bn, n_rows, n_cols, nthreads=8)
    _check(K.spmm_csc(n_rows, n_cols, _dev(a), B), want)


@pytest.mark.parametrize("ld,offset", [(20003, 0), (20000, 1), (20008, 4)])
def test_spmm_csc_unaligned_b(K, ld, offset):
    """ldb % 4 != 0 or an unaligned base: plain loads instead of bulk copies"""
    rng = np.random.default_rng(7)
    n_rows, n_cols, nnz, k = 10000, 20000, 150000, 20
    a = _case(rng, n_rows, n_cols, rng.integers(0, n_rows, nnz), rng.integers(0, n_cols, nnz))
    B, Bn = _B(rng, n_cols, k, ld=ld, offset=offset)
    want = oracle.spmm(*a, Bn, n_rows, n_cols, nthreads=8)
    _check(K.spmm_csc(n_rows, n_cols, _dev(a), B), want)


def test_spmm_csc_heavy_and_hypersparse(K):
    """one column holding 30k entries (spans 15 tiles), a run of 1-entry
    columns (a tile spanning > 512 columns: global-memory path), empty
    columns, and a short tail tile"""
    rng = np.random.default_rng(9)
    n_rows, n_cols = 40000, 60000
    rows = [rng.integers(0, n_rows, 30000), rng.integers(0, n_rows, 20000), rng.integers(0, n_rows, 50003)]
    cols = [np.full(30000, 17), np.arange(100, 40100, 2), rng.integers(50000, 52000, 50003)]
    a = _case(rng, n_rows, n_cols, np.concatenate(rows), np.concatenate(cols))
    B, Bn = _B(rng, n_cols, 24)
    want = oracle.spmm(*a, Bn, n_rows, n_cols, nthreads=8)
    _check(K.spmm_csc(n_rows, n_cols, _dev(a), B), want)


@pytest.mark.parametrize("n_rows,n_cols", [(0, 10), (10, 0), (7, 9)])
def test_spmm_csc_empty(K, n_rows, n_cols):
    a = (np.zeros(0), np.zeros(0, np.int64), np.zeros(n_cols + 1, np.int64))
    B = torch.ones((max(n_cols, 0), 3), dtype=torch.float32, device=DEV).t().contiguous().t()
    C = K.spmm_csc(n_rows, n_cols, _dev(a), B)
    assert C.shape == (n_rows, 3) and not torch.any(C != 0)


def test_spmat_first_product_by_columns():
    """SpMat @ X on a fresh CSC: the first product runs the column merge (no
    CSR built), the second builds and uses the CSR; both match the oracle,
    and a write to the matrix resets the choice"""
    from paper_1805_03380_b200 import SpMat, CscData, Dims

    rng = np.random.default_rng(12)
    n_rows, n_cols, nnz, k = 20000, 15000, 150000, 32
    a = _case(rng, n_rows, n_cols, rng.integers(0, n_rows, nnz), rng.integers(0, n_cols, nnz))
    p, r, v = _dev(a)
    m = SpMat.from_csc(CscData(Dims(n_rows, n_cols), p, r, v))
    B, Bn = _B(rng, n_cols, k)
    want = oracle.spmm(*a, Bn, n_rows, n_cols, nthreads=8)
    C1 = m @ B
    assert m._csr is None and m._csc_mm == 1
    _check(C1, want)
    C2 = m @ B
    assert m._csr is not None
    _check(C2, want)
