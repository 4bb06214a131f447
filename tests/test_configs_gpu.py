"""Parity at the full BASELINE.json configuration sizes (seeded synthetic
inputs, paper_1805_03380_b200.synth): every device result against the CPU
oracle on the same inputs -- structure bit-exact, values bit-exact where the
reference order is reproduced, float32 SpMM within 1e-5, trace within 1e-12
-- plus size-independent properties (involution, commutativity, Frobenius)."""

import numpy as np
import pytest
import torch

import oracle
from conftest import assert_close, assert_csc_equal
from paper_1805_03380_b200 import Dims, SpMat, _kernels, synth
from paper_1805_03380_b200 import csc as csc_mod

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def T(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def dev_csc(v, r, o, vdt=torch.float64):
    return T(o, torch.int32), T(r, torch.int32), T(v, vdt)


def host(c):
    p, r, v = c
    return v.cpu().numpy().astype(np.float64), r.cpu().numpy(), p.cpu().numpy()


def test_cfg1_build_and_transpose():
    n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
    m = SpMat.from_triplets(n_rows, n_cols, (rows, cols, vals))
    want = oracle.canonicalize(n_rows, n_cols, rows, cols, vals)
    got = m.csc()
    assert got.nnz == 995_078
    assert_csc_equal((got.values, got.row_indices, got.col_offsets), want, exact_values=True)
    t = m.t().csc()
    assert_csc_equal((t.values, t.row_indices, t.col_offsets), oracle.transpose(n_rows, n_cols, *want),
                     exact_values=True)
    assert m.t().t().csc().same_elements(got)


def test_cfg2_incremental_writes_and_flush():
    n, _, rows, cols, vals = synth.cfg2_writes()
    m = SpMat.zeros(n, n)
    for i in range(rows.shape[0]):  # element-wise API, as the reference's workload
        m[int(rows[i]), int(cols[i])] = float(vals[i])
    got = m.csc()
    want = oracle.flush(n, n, (np.empty(0), np.empty(0, np.int64), np.zeros(n + 1, np.int64)), rows, cols, vals)
    assert got.nnz == 190_000
    assert_csc_equal((got.values, got.row_indices, got.col_offsets), want, exact_values=True)


def test_cfg3_spmm_f32():
    n, _, av, ar, ao, B = synth.cfg3_spmm()
    A = dev_csc(av, ar, ao, torch.float32)
    csr = _kernels.transpose(n, n, *A)
    Bd = torch.as_tensor(B.T.copy(), device="cuda").t()
    C = _kernels.spmm(n, n, csr, Bd).cpu().numpy().astype(np.float64)
    # oracle on every one of the 64 dense columns (each one mat_times_vec of
    # float64 upcasts, _kernels.py:118-127)
    want = oracle.spmm(av.astype(np.float64), ar, ao, B.astype(np.float64), n, n, nthreads=16)
    assert np.all(np.abs(C - want) <= 1e-5 * np.maximum(1.0, np.abs(want)))
    Ce = _kernels.spmm(n, n, csr, Bd, exact=True).cpu().numpy().astype(np.float64)
    assert np.array_equal(Ce, want.astype(np.float32).astype(np.float64))
    # column merge straight over the CSC (the first product on a fresh handle)
    Cm = _kernels.spmm_csc(n, n, A, Bd).cpu().numpy().astype(np.float64)
    assert np.all(np.abs(Cm - want) <= 1e-5 * np.maximum(1.0, np.abs(want)))


def test_cfg4_trace():
    n, _, A, B = synth.cfg4_trace_pair()
    got = float(_kernels.fused_trace(n, n, dev_csc(*A), dev_csc(*B))[0].item())
    want = oracle.fused_trace(n, *A, *B)
    assert want == -6.0515221450266097  # SURVEY 6.2 / Appendix A, seeds 4 / 40 (9,976 matches)
    assert_close(got, want)
    fro = float(_kernels.fused_trace(n, n, dev_csc(*A), dev_csc(*A))[0].item())
    assert_close(fro, float(np.sum(A[0] * A[0])), tol=1e-12)


def test_cfg5_add_and_spgemm():
    n, _, A, B = synth.cfg5_pair()
    assert (A[2][-1], B[2][-1]) == (3_258_067, 3_182_595)
    assert int(np.diff(A[2])[B[1]].sum()) == 51_847_707  # Gustavson products
    a, b = dev_csc(*A), dev_csc(*B)
    add = host(_kernels.linear_combine(n, n, a, b, 1.0, 1.0))
    assert_csc_equal(add, oracle.linear_combine(n, *A, *B, 1.0, 1.0), exact_values=True)
    add2 = host(_kernels.linear_combine(n, n, b, a, 1.0, 1.0))
    assert_csc_equal(add2, add, exact_values=True)  # commutative bit for bit
    C = host(_kernels.spgemm(n, n, n, a, b))
    assert_csc_equal(C, oracle.spgemm(n, *A, *B, n), exact_values=True)
