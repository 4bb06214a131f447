"""Run one hot-path op a few times on its BASELINE config (for ncu captures).

    python tools/op_runner.py build|flush|transpose|spmm|trace|add|spgemm|all [reps]

`all` runs every op in that order, `reps` times each, in one process (one
ncu capture for the whole set).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import SpMat, _kernels, synth  # noqa: E402
from paper_1805_03380_b200.csc import CscData, Dims  # noqa: E402


def main():
    op = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    for o in (("build", "transpose", "flush", "spmm", "spmm_first", "trace", "add", "spgemm", "build_1e7",
               "transpose_1e7_f32") if op == "all" else (op,)):
        run(o, reps)


def rng_(op):
    """NVTX range around one call of the op: `ncu --nvtx --nvtx-include
    op_<name>/` then captures exactly the launches of that call
    (tools/ncu_ops.sh), so per-op DRAM traffic is summed over all of them."""
    return torch.cuda.nvtx.range("op_" + op)


def run(op, reps):
    dev = torch.device("cuda")

    def T(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    if op in ("build", "transpose"):
        n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
        r, c, v = T(rows, torch.int32), T(cols, torch.int32), T(vals, torch.float64)
        p, ri, vv, _ = _kernels.coo_to_csc(n_rows, n_cols, r, c, v)
        for _ in range(reps):
            with rng_(op):
                if op == "build":
                    _kernels.coo_to_csc(n_rows, n_cols, r, c, v)
                else:
                    _kernels.transpose(n_rows, n_cols, p, ri, vv)
    elif op == "flush":
        n, _, rows, cols, vals = synth.cfg2_writes()
        base = (torch.zeros(n + 1, dtype=torch.int32, device=dev), torch.empty(0, dtype=torch.int32, device=dev),
                torch.empty(0, dtype=torch.float64, device=dev))
        lr, lc, lv = T(rows, torch.int32), T(cols, torch.int32), T(vals, torch.float64)
        for _ in range(reps):
            with rng_(op):
                _kernels.flush_log(n, n, base, lr, lc, lv)
    elif op in ("spmm", "spmm_first"):
        n, _, av, ar, ao, B = synth.cfg3_spmm()
        a = (T(ao, torch.int32), T(ar, torch.int32), T(av, torch.float32))
        csr = _kernels.transpose(n, n, *a)
        Bd = torch.as_tensor(B.T.copy(), device=dev).t()
        for _ in range(reps):
            with rng_(op):
                if op == "spmm":
                    _kernels.spmm(n, n, csr, Bd)
                else:  # first product on a fresh CSC handle: its CSR conversion is part of the op
                    SpMat.from_csc(CscData(Dims(n, n), *a)) @ Bd
    elif op in ("build_1e7", "transpose_1e7_f32"):  # large-input pipeline (bench.py bench_large_n)
        n = 1_000_000
        g = torch.Generator(device=dev)
        g.manual_seed(7)
        vdt = torch.float64 if op == "build_1e7" else torch.float32
        rows = torch.randint(0, n, (10_000_000,), device=dev, dtype=torch.int32, generator=g)
        cols = torch.randint(0, n, (10_000_000,), device=dev, dtype=torch.int32, generator=g)
        vals = (torch.rand(10_000_000, device=dev, dtype=torch.float64, generator=g) * 2 - 1).to(vdt)
        p, ri, vv, _ = _kernels.coo_to_csc(n, n, rows, cols, vals)
        for _ in range(reps):
            with rng_(op):
                if op == "build_1e7":
                    _kernels.coo_to_csc(n, n, rows, cols, vals)
                else:
                    _kernels.transpose(n, n, p, ri, vv)
    elif op in ("trace", "add", "spgemm"):
        if op == "trace":
            n, _, A, B = synth.cfg4_trace_pair()
        else:
            n, _, A, B = synth.cfg5_pair()
        a = (T(A[2], torch.int32), T(A[1], torch.int32), T(A[0], torch.float64))
        b = (T(B[2], torch.int32), T(B[1], torch.int32), T(B[0], torch.float64))
        for _ in range(reps):
            with rng_(op):
                if op == "trace":
                    _kernels.fused_trace(n, n, a, b)
                elif op == "add":
                    _kernels.linear_combine(n, n, a, b, 1.0, 1.0)
                else:
                    _kernels.spgemm(n, n, n, a, b)
    torch.cuda.synchronize()
    print("ok", op)


if __name__ == "__main__":
    main()
