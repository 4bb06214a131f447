"""The C ABI's multi-GPU entry points (include/bsparse.h as_mg_*, csrc/mg.cu):
the rank-local kernel + its NCCL collective in one call, on a communicator the
caller owns.  One GPU is all this environment reaches, so the communicator has
one rank (created here with NCCL's own C API through ctypes); the column ranges
of a two-rank split are run one after the other and combined as the ranks'
all-gather would (dist.dd_combine, rank order).  Oracle: the single-GPU result
and oracle.fused_trace (_kernels.py:153-175), 1e-12; SpMM blocks bit-identical
to the single-GPU kernel."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_close

pytestmark = pytest.mark.gpu


class _UniqueId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_byte * 128)]


@pytest.fixture(scope="module")
def K():
    from paper_1805_03380_b200 import _kernels

    return _kernels


@pytest.fixture(scope="module")
def comm(K):
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    try:
        nccl = ctypes.CDLL("libnccl.so.2")  # the copy torch has loaded
    except OSError:
        pytest.skip("no libnccl.so.2 in this process")
    nccl.ncclGetUniqueId.argtypes = [ctypes.POINTER(_UniqueId)]
    nccl.ncclCommInitRank.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, _UniqueId, ctypes.c_int]
    nccl.ncclCommDestroy.argtypes = [ctypes.c_void_p]
    uid = _UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    c = ctypes.c_void_p()
    assert nccl.ncclCommInitRank(ctypes.byref(c), 1, uid, 0) == 0
    K.mg_init(c.value, 0, 1)
    yield c
    K.mg_shutdown()
    nccl.ncclCommDestroy(c)


def _rand_csc(seed, n_rows, n_cols, n):
    g = np.random.default_rng(seed)
    return oracle.canonicalize(n_rows, n_cols, g.integers(0, n_rows, n), g.integers(0, n_cols, n), g.uniform(-1, 1, n))


def _dev(c, vdt=torch.float64):
    vals, rows, offs = c
    return (torch.as_tensor(np.ascontiguousarray(offs, dtype=np.int32), device="cuda"),
            torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int32), device="cuda"),
            torch.as_tensor(np.ascontiguousarray(vals), device="cuda").to(vdt))


def test_not_initialised_is_an_argument_error():
    from paper_1805_03380_b200 import _lib

    L = _lib.lib()
    _lib.check(L.as_mg_shutdown())
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    rc = L.as_mg_trace_atb_f64(4, 4, None, None, None, None, None, None, 0, 0, 0, 4, _lib.ptr(out), None, 0, None)
    assert rc == 5  # AS_ERR_ARG
    assert b"as_mg_init" in L.as_last_error()


@pytest.mark.parametrize("n_rows,n_cols,n", [(50_000, 20_000, 2_000_000), (3000, 501, 40_000)])
def test_trace_over_column_ranges(K, comm, n_rows, n_cols, n):
    from paper_1805_03380_b200 import dist as D

    a, b = _rand_csc(1, n_rows, n_cols, n), _rand_csc(2, n_rows, n_cols, n)
    want = oracle.fused_trace(n_cols, *a, *b)
    da, db = _dev(a), _dev(b)
    whole = K.mg_fused_trace(n_rows, n_cols, da, db, 0, n_cols).cpu().numpy()
    single = K.fused_trace(n_rows, n_cols, da, db).cpu().numpy()
    assert_close(float(whole[0]), want)
    assert float(whole[0]) == float(single[0])
    # the two ranks of a split, one after the other, combined in rank order
    bounds = D.split_by_weight(np.diff(a[2]) + np.diff(b[2]), 2)
    parts = [K.mg_fused_trace(n_rows, n_cols, da, db, int(bounds[r]), int(bounds[r + 1])).cpu().tolist()
             for r in range(2)]
    assert_close(D.dd_combine(parts), want)
    # empty range
    assert K.mg_fused_trace(n_rows, n_cols, da, db, 7, 7).cpu().tolist() == [0.0, 0.0]


def test_trace_range_outside_the_matrix(K, comm):
    from paper_1805_03380_b200.errors import ShapeError

    a = _dev(_rand_csc(3, 100, 50, 500))
    with pytest.raises(ShapeError):
        K.mg_fused_trace(100, 50, a, a, 10, 51)


@pytest.mark.parametrize("k", [1, 16, 24])
def test_spmm_block_gather(K, comm, k):
    n_rows, n_cols = 4000, 3000
    a = _rand_csc(4, n_rows, n_cols, 60_000)
    at = oracle.transpose(n_rows, n_cols, *a)
    csr = _dev(at, torch.float32)
    X = torch.randn(k, n_cols, device="cuda").t()  # column-major (n_cols, k)
    want = K.spmm(n_rows, n_cols, csr, X)
    got = K.mg_spmm(n_rows, n_cols, csr, X)
    assert torch.equal(got, want)


def test_spgemm_slices_stay_distributed(K, comm):
    from paper_1805_03380_b200 import dist as D

    m, kk, n = 900, 700, 800
    a, b = _rand_csc(5, m, kk, 9000), _rand_csc(6, kk, n, 8000)
    want = oracle.spgemm(m, *a, *b, n)
    da = _dev(a)
    # the two ranks' column slices of B, one after the other (each a one-rank gather)
    bounds = [0, 350, n]
    got_vals, got_rows, got_ptr = [], [], [0]
    for r in range(2):
        c0, c1 = bounds[r], bounds[r + 1]
        sl = D.csc_column_slice(np.asarray(b[2]), np.asarray(b[1]), np.asarray(b[0]), c0, c1)  # (ptr, rows, vals)
        db = _dev((sl[2], sl[1], sl[0]))
        p, ri, v, snnz, soff = K.mg_spgemm(m, kk, c1 - c0, da, db)
        assert snnz.cpu().tolist() == [int(ri.shape[0])] and soff.cpu().tolist() == [0]
        got_vals.append(v.cpu().numpy())
        got_rows.append(ri.cpu().numpy())
        got_ptr.extend((p.cpu().numpy()[1:].astype(np.int64) + got_ptr[-1]).tolist())
    assert np.array_equal(np.asarray(got_ptr), want[2])
    assert np.array_equal(np.concatenate(got_rows), want[1])
    assert np.array_equal(np.concatenate(got_vals).view(np.int64), want[0].view(np.int64))
