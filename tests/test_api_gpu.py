"""The reference's own hot-path tests, re-run through this
package's SpMat API on the GPU: construction pins (test_csc.py:18-59),
COO interchange (test_coo.py:35-65), insertion / flush semantics and
conversion counters (test_hybrid.py:100-226), transpose / add / SpGEMM / SpMV
against a dense shadow (test_ops.py), fused trace and temporaries
(test_expr.py:132-178) and the Fig. 1 scenario (test_acceptance.py:330-353)."""

import numpy as np
import pytest
import torch

import oracle
from conftest import TOL64, assert_close
from paper_1805_03380_b200 import (Add, CoordinateError, CorruptionError, Dims, Format, Mul, ScalarMul, ShapeError,
                                   SpMat, Trace, Transpose, evaluate, evaluate_counting, fused_trace_at_b, lift, ops)
from paper_1805_03380_b200 import coo as coo_mod
from paper_1805_03380_b200 import csc as csc_mod

pytestmark = pytest.mark.gpu


def dense_triplets(d):
    out = []
    for c in range(d.shape[1]):
        for r in range(d.shape[0]):
            if d[r, c] != 0.0:
                out.append((r, c, float(d[r, c])))
    return out


def random_dense(rng, r, c, density):
    d = np.zeros((r, c))
    k = int(round(density * r * c))
    if k:
        pos = rng.choice(r * c, size=min(k, r * c), replace=False)
        vals = rng.uniform(-1, 1, size=pos.shape[0])
        vals[vals == 0.0] = 0.5
        d[pos % r, pos // r] = vals
    return d


def make_pair(rng, r, c, density):
    d = random_dense(rng, r, c, density)
    return SpMat.from_triplets(r, c, dense_triplets(d)), d


def assert_matches_dense(m, dense, tol=TOL64):
    data = m.csc() if isinstance(m, SpMat) else m
    csc_mod.validate(data)
    assert data.dims == Dims(dense.shape[0], dense.shape[1])
    got = [(t.row, t.col) for t in data.triplets()]
    want = [(r, c) for r, c, _ in dense_triplets(dense)]
    assert got == want
    for t in data.triplets():
        ref = dense[t.row, t.col]
        assert abs(t.value - ref) <= tol * max(1.0, abs(ref))


# -- construction (test_csc.py:18-59) ---------------------------------------------
def test_example_and_edge_pins():
    m = csc_mod.from_triplets(Dims(3, 2), [(0, 0, 1.0), (2, 1, 3.0), (1, 1, 2.0)])
    assert m.values.tolist() == [1.0, 2.0, 3.0] and m.row_indices.tolist() == [0, 1, 2]
    assert m.col_offsets.tolist() == [0, 1, 3]
    e = csc_mod.from_triplets(Dims(4, 4), [])
    assert e.nnz == 0 and e.col_offsets.tolist() == [0, 0, 0, 0, 0]
    assert csc_mod.from_triplets(Dims(2, 2), [(0, 0, 5.0), (0, 0, -5.0)]).nnz == 0
    assert csc_mod.from_triplets(Dims(2, 2), [(1, 0, 2.0), (1, 0, 3.0)]).get(1, 0) == 5.0
    lw = csc_mod.from_triplets(Dims(2, 2), [(1, 0, 2.0), (0, 1, 9.0), (1, 0, 3.0)], csc_mod.DUP_LAST)
    assert lw.get(1, 0) == 3.0 and lw.get(0, 1) == 9.0
    with pytest.raises(CoordinateError, match="triplet 1"):
        csc_mod.from_triplets(Dims(2, 2), [(0, 0, 1.0), (5, 0, 2.0)])


def test_random_roundtrips(rng):
    for _ in range(50):
        r, c = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        dense = random_dense(rng, r, c, 0.3)
        m = csc_mod.from_triplets(Dims(r, c), dense_triplets(dense))
        csc_mod.validate(m)
        assert np.array_equal(m.to_dense(), dense)


def test_coo_interchange(rng):
    m = csc_mod.from_triplets(Dims(5, 4), [(4, 3, 1.0), (0, 0, 2.0), (4, 3, 1.5), (2, 1, -1.0), (2, 1, 1.0)])
    assert m.nnz == 2 and m.get(4, 3) == 2.5
    coo = coo_mod.from_csc(m)
    assert coo_mod.to_csc(coo).same_elements(m)
    bad = coo_mod.CooData(Dims(2, 2), [0, 3], [0, 0], [1.0, 1.0])
    with pytest.raises(CorruptionError):
        coo_mod.to_csc(bad)


# -- insertion cache / flush (test_hybrid.py:100-226) -------------------------------
def test_overwrite_fast_path_keeps_csc(rng):
    m, _ = make_pair(rng, 8, 8, 0.5)
    t = next(iter(m.triplets()))
    m.set(t.row, t.col, 42.0)
    assert m.valid_formats == {Format.CSC} and m.conversions[Format.RBT] == 0
    assert m.get(t.row, t.col) == 42.0
    assert m.csc().vals[m.csc().find(t.row, t.col)].item() == 42.0


def test_structural_write_and_erase(rng):
    dense = random_dense(rng, 8, 8, 0.2)
    dense[5, 5] = 0.0
    m = SpMat.from_triplets(8, 8, dense_triplets(dense))
    m.set(5, 5, 3.25)
    assert m.valid_formats == {Format.RBT} and m.conversions[Format.RBT] == 1
    assert m.get(5, 5) == 3.25
    n = m.nnz
    m.set(5, 5, 0.0)
    assert m.nnz == n - 1 and m.get(5, 5) == 0.0


def test_random_writes_match_batch_of_final_state(rng):
    dense = random_dense(rng, 20, 20, 0.15)
    m = SpMat.from_triplets(20, 20, dense_triplets(dense))
    for _ in range(1000):
        i, j = int(rng.integers(0, 20)), int(rng.integers(0, 20))
        v = float(rng.integers(0, 4))
        m.set(i, j, v)
        dense[i, j] = v
    batch = SpMat.from_triplets(20, 20, dense_triplets(dense))
    assert m.csc().same_elements(batch.csc())
    assert m.conversions[Format.CSC] == 1


def test_accumulate_shadow(rng):
    dense = np.zeros((15, 15))
    m = SpMat.zeros(15, 15)
    for _ in range(500):
        i, j = int(rng.integers(0, 15)), int(rng.integers(0, 15))
        d = float(rng.uniform(-1, 1))
        m.accumulate(i, j, d)
        dense[i, j] += d
    assert_matches_dense(m, dense)


def test_batch_insert_merges_by_sum():
    m = SpMat.from_triplets(3, 3, [(0, 0, 2.0), (1, 1, 1.0)])
    m.batch_insert([(0, 0, 3.0), (2, 2, 7.0), (1, 1, -1.0)])
    assert m.get(0, 0) == 5.0 and m.get(2, 2) == 7.0 and m.get(1, 1) == 0.0
    assert m.valid_formats == {Format.CSC}


def test_set_many_matches_reference_flush(rng):
    r, c = 300, 200
    base = oracle.canonicalize(r, c, rng.integers(0, r, 2000), rng.integers(0, c, 2000), rng.uniform(-1, 1, 2000))
    m = SpMat.from_csc(csc_mod.CscData.from_reference_arrays(Dims(r, c), *base))
    wr, wc = rng.integers(0, r, 20000), rng.integers(0, c, 20000)
    wv = rng.uniform(-1, 1, 20000)
    wv[rng.random(20000) < 0.1] = 0.0
    m.set_many(wr, wc, wv)
    want = oracle.flush(r, c, base, wr, wc, wv)
    got = m.csc()
    assert np.array_equal(got.col_offsets, want[2]) and np.array_equal(got.row_indices, want[1])
    assert np.array_equal(got.values, want[0])


# -- operations (test_ops.py) ----------------------------------------------------------
def test_add_subtract_vs_dense(rng):
    for _ in range(30):
        r, c = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        a, da = make_pair(rng, r, c, 0.2)
        b, db = make_pair(rng, r, c, 0.2)
        assert_matches_dense(a + b, da + db)
        assert_matches_dense(a - b, da - db)
    a, _ = make_pair(rng, 10, 8, 0.3)
    assert ops.subtract(a, a).nnz == 0
    with pytest.raises(ShapeError):
        ops.add(Z3x4(), Z4x3())


def Z3x4():
    return SpMat.zeros(3, 4)


def Z4x3():
    return SpMat.zeros(4, 3)


def test_matmul_vs_dense(rng):
    for _ in range(25):
        m, k, n = (int(rng.integers(1, 50)) for _ in range(3))
        a, da = make_pair(rng, m, k, 0.2)
        b, db = make_pair(rng, k, n, 0.2)
        assert_matches_dense(a @ b, da @ db)
    a = SpMat.from_triplets(10, 10, [(2, 5, 1.0), (3, 7, 1.0)])
    b = SpMat.from_triplets(10, 10, [(5, 0, 2.0), (7, 1, 3.0)])
    out = a @ b
    assert out.nnz == 2 and out.get(2, 0) == 2.0 and out.get(3, 1) == 3.0
    i8 = ops.speye(8, 8)
    a, da = make_pair(rng, 8, 8, 0.3)
    assert_matches_dense(i8 @ a, da)
    assert_matches_dense(a @ i8, da)


def test_transpose_vs_dense_and_law(rng):
    for _ in range(25):
        r, c = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        a, da = make_pair(rng, r, c, 0.25)
        assert_matches_dense(a.t(), da.T)
        assert_matches_dense(a.t().t(), da)
    a, _ = make_pair(rng, 12, 9, 0.3)
    b, _ = make_pair(rng, 9, 14, 0.3)
    assert (a @ b).t().csc().same_elements((b.t() @ a.t()).csc()) or np.allclose(
        (a @ b).t().to_dense(), (b.t() @ a.t()).to_dense(), rtol=0, atol=1e-12)


def test_spmv_and_spmm(rng):
    for _ in range(20):
        r, c = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        a, da = make_pair(rng, r, c, 0.2)
        v, x = rng.random(r), rng.random(c)
        assert np.all(np.abs(ops.vec_times_mat(v, a) - v @ da) <= 1e-12 * np.maximum(1.0, np.abs(v @ da)))
        assert np.all(np.abs(a @ x - da @ x) <= 1e-12 * np.maximum(1.0, np.abs(da @ x)))
        assert np.allclose(v @ a, v @ da)
        X = rng.standard_normal((c, 5))
        C = a @ X
        assert C.shape == (r, 5) and np.all(np.abs(C - da @ X) <= 1e-12 * np.maximum(1.0, np.abs(da @ X)))
    with pytest.raises(ShapeError):
        ops.mat_times_vec(SpMat.zeros(3, 5), np.ones(3))


def test_scalar_mul(rng):
    a, da = make_pair(rng, 9, 9, 0.3)
    assert_matches_dense(0.5 * a, 0.5 * da)
    assert ops.scalar_mul(a, 0.0).nnz == 0


# -- expressions (test_expr.py:132-178) ------------------------------------------------
def test_fused_trace_pins(rng):
    a = SpMat.from_triplets(2, 2, [(0, 0, 1.0), (1, 1, 2.0)])
    b = SpMat.from_triplets(2, 2, [(0, 0, 3.0), (1, 1, 4.0)])
    assert fused_trace_at_b(a, b) == 11.0
    a, _ = make_pair(rng, 9, 9, 0.4)
    assert_close(fused_trace_at_b(a, a), ops.norm_fro(a) ** 2)
    assert fused_trace_at_b(SpMat.from_triplets(3, 3, [(0, 0, 5.0)]), SpMat.from_triplets(3, 3, [(1, 1, 7.0)])) == 0.0
    for _ in range(10):
        a, _ = make_pair(rng, 12, 12, 0.3)
        b, _ = make_pair(rng, 12, 12, 0.3)
        e = Trace(Mul(Transpose(lift(a)), lift(b)))
        assert_close(evaluate(e), evaluate(e, optimize=False))
    with pytest.raises(ShapeError):
        fused_trace_at_b(SpMat.zeros(3, 4), SpMat.zeros(4, 3))


def test_temporaries(rng):
    a, _ = make_pair(rng, 10, 10, 0.3)
    b, _ = make_pair(rng, 10, 10, 0.3)
    _, fused = evaluate_counting(Trace(Mul(Transpose(lift(a)), lift(b))), optimize=True)
    _, naive = evaluate_counting(Trace(Mul(Transpose(lift(a)), lift(b))), optimize=False)
    assert fused == 0 and naive == 2
    e = ScalarMul(0.5, Add(lift(a), lift(b)))
    assert evaluate_counting(e, optimize=True)[1] == 0 and evaluate_counting(e, optimize=False)[1] == 1


# -- Fig. 1 scenario (test_acceptance.py:330-353) ------------------------------------------
def test_fig1_scenario():
    x = ops.sprandu(1000, 1000, 0.01, seed=4242)
    shadow = x.to_dense()
    x[1, 1] = 1.23
    shadow[1, 1] = 1.23
    x[3, 4] += 4.56
    shadow[3, 4] += 4.56
    v = np.random.default_rng(7).random(1000)
    w = v @ x
    assert x.conversions[Format.RBT] <= 1 and x.conversions[Format.CSC] <= 1
    want = v @ shadow
    assert np.all(np.abs(w - want) <= TOL64 * np.maximum(1.0, np.abs(want)))


def test_device_tensors_in_and_out():
    rng = np.random.default_rng(3)
    rows = torch.as_tensor(rng.integers(0, 100, 5000), device="cuda")
    cols = torch.as_tensor(rng.integers(0, 80, 5000), device="cuda")
    vals = torch.as_tensor(rng.uniform(-1, 1, 5000), device="cuda")
    m = SpMat.from_triplets(100, 80, (rows, cols, vals))
    X = torch.randn(80, 3, dtype=torch.float64, device="cuda")
    C = m @ X
    assert isinstance(C, torch.Tensor) and C.is_cuda
    want = m.to_dense() @ X.cpu().numpy()
    assert np.allclose(C.cpu().numpy(), want, rtol=0, atol=1e-12)


def test_transposed_operand_reads_the_cached_csr():
    """0.5*(A+B) @ C.t() -- the transpose is read through C's
    cached CSR, not materialised; same result as the naive post-order."""
    from paper_1805_03380_b200 import Add, Mul, ScalarMul, Transpose, evaluate_counting, lift

    rng = np.random.default_rng(11)
    mats = []
    for _ in range(3):
        d = np.where(rng.random((14, 14)) < 0.3, rng.standard_normal((14, 14)), 0.0)
        mats.append(SpMat.from_dense(d, device="cuda"))
    a, b, c = mats
    e = Mul(ScalarMul(0.5, Add(lift(a), lift(b))), Transpose(lift(c)))
    opt, t_opt = evaluate_counting(e, optimize=True)
    naive, t_naive = evaluate_counting(e, optimize=False)
    assert t_opt == 1 and t_naive == 3  # the scaled sum only / sum, scaling and transpose
    assert opt.csc().same_elements(naive.csc())


def test_canonicalize_host_zero_copy():
    """csc.canonicalize_host: pinned host triplets read over PCIe inside the
    build kernel, the CSC written straight into pinned host memory; same
    result as the device path and the oracle, bad triplets reported."""
    import torch

    import oracle
    from paper_1805_03380_b200 import csc as C
    from paper_1805_03380_b200.csc import Dims
    from paper_1805_03380_b200.errors import CoordinateError

    rng = np.random.default_rng(21)
    for (r, c, n) in [(300, 200, 5000), (7, 5, 300), (10000, 10000, 200000), (50, 40, 0)]:
        rows, cols, vals = rng.integers(0, r, n), rng.integers(0, c, n), rng.uniform(-1, 1, n)
        got = C.canonicalize_host(Dims(r, c), rows, cols, vals)
        assert got.col_ptr.device.type == "cpu"
        want = oracle.canonicalize(r, c, rows, cols, vals)
        assert np.array_equal(got.col_offsets, want[2]) and np.array_equal(got.row_indices, want[1])
        assert np.array_equal(got.values.view(np.int64), want[0].view(np.int64))
    rows = np.array([0, 5, 1], dtype=np.int64)
    with pytest.raises(CoordinateError, match="coordinate 1"):
        C.canonicalize_host(Dims(3, 3), rows, np.array([0, 0, 1]), np.array([1.0, 2.0, 3.0]))
    # reused pinned output buffers, LastWins
    out = (torch.empty(4, dtype=torch.int32).pin_memory(), torch.empty(4, dtype=torch.int32).pin_memory(),
           torch.empty(4, dtype=torch.float64).pin_memory())
    m = C.canonicalize_host(Dims(2, 3), np.array([1, 1, 0, 1]), np.array([0, 0, 2, 0]),
                            np.array([2.0, 3.0, 9.0, 4.0]), C.DUP_LAST, out=out)
    assert m.get(1, 0) == 4.0 and m.get(0, 2) == 9.0 and m.nnz == 2


def test_int64_host_upload_narrowing():
    """Host int64 triplets take the narrowing upload (as_upload_coo_i64):
    pinned and pageable inputs, chunk edges, and indices that do not fit
    int32 (2^32 + r, negatives) reported as the first bad triplet -- the
    same CoordinateError index as the device path."""
    from paper_1805_03380_b200 import _kernels

    rng = np.random.default_rng(77)
    for (r, c, n) in [(300, 200, 5000), (7, 5, 1), (10000, 10000, 300001), (50, 40, 0)]:
        rows, cols, vals = rng.integers(0, r, n), rng.integers(0, c, n), rng.uniform(-1, 1, n)
        want = oracle.canonicalize(r, c, rows, cols, vals)
        for pinned in (False, True):
            args = (rows, cols, vals)
            if pinned:
                args = tuple(torch.from_numpy(a).pin_memory() for a in args)
            m = SpMat.from_triplets(r, c, args).csc()
            assert np.array_equal(m.col_offsets, want[2]) and np.array_equal(m.row_indices, want[1])
            assert np.array_equal(m.values.view(np.int64), want[0].view(np.int64))
    # direct: narrowed indices, -1 for anything outside [0, 2^31)
    rows = np.array([3, (1 << 32) + 3, -5, (1 << 31) - 1, 1 << 31], dtype=np.int64)
    d_r, d_c, d_v = _kernels.upload_coo(torch.from_numpy(rows), torch.from_numpy(rows.copy()),
                                        torch.arange(5, dtype=torch.float64))
    assert d_r.cpu().tolist() == [3, -1, -1, (1 << 31) - 1, -1] and d_c.cpu().tolist() == d_r.cpu().tolist()
    assert d_v.cpu().tolist() == [0.0, 1.0, 2.0, 3.0, 4.0]
    for bad_pos, bad_val in [(2, (1 << 32) + 1), (4, -1), (0, 1 << 40)]:
        rows = np.zeros(6, dtype=np.int64)
        rows[bad_pos] = bad_val
        with pytest.raises(CoordinateError, match="triplet %d " % bad_pos):
            SpMat.from_triplets(4, 4, (rows, np.zeros(6, dtype=np.int64), np.ones(6)))


def test_packed_key_upload():
    """Shapes whose row + column bit widths fit 31 bits move one 32-bit key per
    triplet (as_upload_coo_packed); coordinates outside the shape (not just
    outside int32) arrive as -1; wider shapes keep the int32 pair upload."""
    from paper_1805_03380_b200 import _kernels

    nr, nc = 1 << 16, 1 << 15  # 16 + 15 bits: the largest key is 0x7fffffff
    rows = np.array([0, nr - 1, nr, -1, 5, nr - 1], dtype=np.int64)
    cols = np.array([0, nc - 1, 0, 0, nc, 3], dtype=np.int64)
    d_r, d_c, _ = _kernels.upload_coo(torch.from_numpy(rows), torch.from_numpy(cols),
                                      torch.arange(6, dtype=torch.float64), shape=(nr, nc))
    assert d_r.cpu().tolist() == [0, nr - 1, -1, -1, -1, nr - 1]
    assert d_c.cpu().tolist() == [0, nc - 1, -1, -1, -1, 3]
    rng = np.random.default_rng(78)
    for (r, c, n) in [(nr, nc, 200000), (1 << 20, 1 << 20, 100000), (1, 1, 10), (3, 1 << 22, 1000)]:
        rows, cols, vals = rng.integers(0, r, n), rng.integers(0, c, n), rng.uniform(-1, 1, n)
        want = oracle.canonicalize(r, c, rows, cols, vals)
        m = SpMat.from_triplets(r, c, (rows, cols, vals)).csc()
        assert np.array_equal(m.col_offsets, want[2]) and np.array_equal(m.row_indices, want[1])
        assert np.array_equal(m.values.view(np.int64), want[0].view(np.int64))
    rows = np.zeros(9, dtype=np.int64)
    rows[6] = 4  # == n_rows: inside int32, outside the shape
    with pytest.raises(CoordinateError, match="triplet 6 "):
        SpMat.from_triplets(4, 4, (rows, np.zeros(9, dtype=np.int64), np.ones(9)))


def test_rbt_snapshot_not_aliased_by_in_place_patch():
    """an RbtStore taken from a SpMat (rbt.from_csc, rbt.py:461-476)
    is an independent store in the reference; a later in-place overwrite of
    a stored value through the SpMat (hybrid.py:170-178) must not show in it."""
    from paper_1805_03380_b200.cache import encode_index

    m = SpMat.from_triplets(4, 3, [(0, 0, 1.0), (2, 1, 3.0), (1, 2, 2.0)])
    t = m.rbt()
    m.set(2, 1, 7.5)  # stored nonzero, CSC valid: patched in place
    assert m.get(2, 1) == 7.5
    assert t.get(encode_index(2, 1, 4)) == 3.0
    assert m.csc().values.tolist() == [1.0, 7.5, 2.0]


@pytest.mark.parametrize("nr,nc,n", [(10000, 10000, 300000), (65536, 8, 70000), (65537, 8, 70000),
                                     (300, 2, 5000), (1 << 20, 3, 100000)])
def test_to_host_read_back(nr, nc, n):
    """CscData.to_host (the e2e read-back): rows of a matrix with <= 65536 rows
    come back at half width and are widened on host threads; the copied
    col_ptr / rows / values equal the device arrays, also from a pending
    (lazily sized) build and into caller-provided pinned buffers."""
    rng = np.random.default_rng(nr + n)
    rows, cols, vals = rng.integers(0, nr, n), rng.integers(0, nc, n), rng.uniform(-1, 1, n)
    rows[0], cols[0] = nr - 1, nc - 1
    want = oracle.canonicalize(nr, nc, rows, cols, vals)
    for out in (None, "pinned"):
        h = tuple(torch.from_numpy(x).pin_memory() for x in (rows, cols, vals))
        data = SpMat.from_triplets(nr, nc, h).csc()
        if out == "pinned":
            out = (torch.empty(nc + 1, dtype=torch.int32).pin_memory(), torch.empty(n, dtype=torch.int32).pin_memory(),
                   torch.empty(n, dtype=torch.float64).pin_memory())
        p, r, v = data.to_host(out=out)
        assert np.array_equal(p.numpy(), want[2]) and np.array_equal(r.numpy(), want[1])
        assert np.array_equal(v.numpy().view(np.int64), want[0].view(np.int64))
        assert torch.equal(data.row_idx.cpu(), r) and data.nnz == r.shape[0]
