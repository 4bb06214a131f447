"""Multi-rank (world size 2, gloo, CPU) tests of the column-sharded trace,
SpMM and SpGEMM drivers in paper_1805_03380_b200.dist.  The per-rank local
kernels are the CPU oracle here (the GPU kernels are covered by the gpu
tests); what is tested is the partitioning, the exchange and the
reassembly, against the single-process oracle result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1805_03380_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rand_csc(rng, n_rows, n_cols, n, zipf=False):
    if zipf:
        lens = np.minimum(rng.zipf(1.5, n_cols), n_rows)
        cols = np.repeat(np.arange(n_cols), lens)
        rows = rng.integers(0, n_rows, cols.shape[0])
    else:
        rows, cols = rng.integers(0, n_rows, n), rng.integers(0, n_cols, n)
    return oracle.canonicalize(n_rows, n_cols, rows, cols, rng.standard_normal(rows.shape[0]))


def _oracle_trace_local(n_rows, n_cols, a, b):
    va, ra, pa = a[2], a[1], a[0]
    vb, rb, pb = b[2], b[1], b[0]
    t = oracle.fused_trace(n_cols, va, ra, pa, vb, rb, pb)
    return [t, 0.0]


def _oracle_spmm_local(n_rows, n_cols, csr, X):
    # csr = (row_ptr, col_idx, vals) of A: transpose back to CSC for the oracle
    rp, ci, v = (np.asarray(x) for x in csr)
    csc = oracle.transpose(n_cols, n_rows, v, ci, rp)
    return torch.from_numpy(oracle.spmm(csc[0], csc[1], csc[2], np.asarray(X), n_rows, n_cols))


def _oracle_spgemm_local(n_rows_a, n_inner, n_cols_b, a, b):
    v, r, p = oracle.spgemm(n_rows_a, a[2], a[1], a[0], b[2], b[1], b[0], n_cols_b)
    return p, r, v


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        n_rows, n_cols = 400, 300
        A = _rand_csc(rng, n_rows, n_cols, 9000)
        B = _rand_csc(rng, n_rows, n_cols, 9000)
        a = (A[2], A[1], A[0])
        b = (B[2], B[1], B[0])
        t = D.dist_fused_trace(n_rows, n_cols, a, b, local=_oracle_trace_local)
        # SpMM over 5 dense columns (uneven split)
        X = rng.standard_normal((n_cols, 5))
        At = oracle.transpose(n_rows, n_cols, *A)
        C = D.dist_spmm(n_rows, n_cols, (At[2], At[1], At[0]), X, local=_oracle_spmm_local)
        # SpGEMM with skewed columns
        Z1 = _rand_csc(rng, 200, 150, 0, zipf=True)
        Z2 = _rand_csc(rng, 150, 180, 0, zipf=True)
        z1, z2 = (Z1[2], Z1[1], Z1[0]), (Z2[2], Z2[1], Z2[0])
        P = D.dist_spgemm(200, 150, 180, z1, z2, local=_oracle_spgemm_local, dst=world - 1)
        # left distributed: this rank's slice with its device-side global offset
        Dc = D.dist_spgemm(200, 150, 180, z1, z2, local=_oracle_spgemm_local, dst=None)
        dslice = (Dc.c0, Dc.c1, Dc.global_col_ptr().numpy(), np.asarray(Dc.row_idx), np.asarray(Dc.vals))
        # C gathered on one rank by point-to-point transfers (uneven column blocks)
        C1 = D.dist_spmm(n_rows, n_cols, (At[2], At[1], At[0]), X, local=_oracle_spmm_local, dst=0)
        # equal blocks: one all_gather_into_tensor
        X4 = rng.standard_normal((n_cols, 4 * world))
        C4 = D.dist_spmm(n_rows, n_cols, (At[2], At[1], At[0]), X4, local=_oracle_spmm_local)
        q.put((rank, t, C.numpy(), P, dslice, None if C1 is None else C1.numpy(), C4.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(400)
@pytest.mark.parametrize("world", [2, 4])
def test_world_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    n_rows, n_cols = 400, 300
    A = _rand_csc(rng, n_rows, n_cols, 9000)
    B = _rand_csc(rng, n_rows, n_cols, 9000)
    want_t = oracle.fused_trace(n_cols, *A, *B)
    X = rng.standard_normal((n_cols, 5))
    want_C = oracle.spmm(*A, X, n_rows, n_cols)
    Z1 = _rand_csc(rng, 200, 150, 0, zipf=True)
    Z2 = _rand_csc(rng, 150, 180, 0, zipf=True)
    want_P = oracle.spgemm(200, *Z1, *Z2, 180)
    X4 = rng.standard_normal((n_cols, 4 * world))
    want_C4 = oracle.spmm(*A, X4, n_rows, n_cols)
    covered = 0
    for rank, t, C, P, dslice, C1, C4 in res:
        assert abs(t - want_t) <= 1e-12 * max(1.0, abs(want_t))
        assert np.array_equal(C, want_C)
        assert np.array_equal(C4, want_C4)
        if rank == 0:
            assert np.array_equal(C1, want_C)
        else:
            assert C1 is None
        if rank == world - 1:
            p, r, v = P
            assert np.array_equal(p, want_P[2]) and np.array_equal(r, want_P[1]) and np.array_equal(v, want_P[0])
        else:
            assert P is None
        c0, c1, gp, r, v = dslice
        assert np.array_equal(gp, want_P[2][c0:c1 + 1])
        s, e = want_P[2][c0], want_P[2][c1]
        assert np.array_equal(r, want_P[1][s:e]) and np.array_equal(v, want_P[0][s:e])
        covered += c1 - c0
    assert covered == 180


def test_split_by_weight_properties():
    rng = np.random.default_rng(1)
    for _ in range(50):
        w = rng.integers(0, 50, rng.integers(1, 200))
        for parts in (1, 2, 3, 8):
            b = D.split_by_weight(w, parts)
            assert b[0] == 0 and b[-1] == len(w) and np.all(np.diff(b) >= 0)
    # Zipf-skewed products split by products, not columns
    w = np.array([1000] + [1] * 999)
    b = D.split_by_weight(w, 2)
    assert b[1] == 1


def test_dd_combine_is_more_accurate_than_naive():
    parts = [(1e16, 0.0), (1.0, 0.0), (-1e16, 0.0)]
    assert D.dd_combine(parts) == 1.0
