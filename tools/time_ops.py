"""Event-timed ops on their BASELINE configs (L2 flushed before every rep),
for comparing build variants:  AS_LIB_PATH=... python tools/time_ops.py add trace [reps]
Prints one line per op: median / min kernel-sequence time in us."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import _kernels, synth  # noqa: E402


def main():
    args = sys.argv[1:]
    reps = int(args[-1]) if args and args[-1].isdigit() else 20
    ops = [a for a in args if not a.isdigit()]
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def T(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    if os.environ.get("AS_TRACE_ENGINE"):
        from paper_1805_03380_b200 import _lib
        _lib.check(_lib.lib().as_set_trace_engine(int(os.environ["AS_TRACE_ENGINE"])))
    for op in ops:
        if op in ("add", "spgemm", "trace", "trace5"):
            n, _, A, B = synth.cfg4_trace_pair() if op == "trace" else synth.cfg5_pair()
            a = (T(A[2], torch.int32), T(A[1], torch.int32), T(A[0], torch.float64))
            b = (T(B[2], torch.int32), T(B[1], torch.int32), T(B[0], torch.float64))
            fn = {"add": lambda: _kernels.linear_combine(n, n, a, b, 1.0, 1.0),
                  "spgemm": lambda: _kernels.spgemm(n, n, n, a, b),
                  "trace": lambda: _kernels.fused_trace(n, n, a, b),
                  "trace5": lambda: _kernels.fused_trace(n, n, a, b)}[op]  # trace on cfg 5's Zipf pair
        elif op in ("build", "transpose"):
            n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
            r, c, v = T(rows, torch.int32), T(cols, torch.int32), T(vals, torch.float64)
            p, ri, vv, _ = _kernels.coo_to_csc(n_rows, n_cols, r, c, v)
            fn = (lambda: _kernels.coo_to_csc(n_rows, n_cols, r, c, v)) if op == "build" else (
                lambda: _kernels.transpose(n_rows, n_cols, p, ri, vv))
        elif op == "flush":
            nf, _, rows, cols, vals = synth.cfg2_writes()
            base = (torch.zeros(nf + 1, dtype=torch.int32, device=dev), torch.empty(0, dtype=torch.int32, device=dev),
                    torch.empty(0, dtype=torch.float64, device=dev))
            r, c, v = T(rows, torch.int32), T(cols, torch.int32), T(vals, torch.float64)
            fn = lambda: _kernels.flush_log(nf, nf, base, r, c, v)  # noqa: E731
        elif op == "spmm":
            n, _, av, ar, ao, Bm = synth.cfg3_spmm()
            csr = _kernels.transpose(n, n, T(ao, torch.int32), T(ar, torch.int32), T(av, torch.float32))
            Bd = torch.as_tensor(Bm.T.copy(), device=dev).t()
            fn = lambda: _kernels.spmm(n, n, csr, Bd)  # noqa: E731
        else:
            raise SystemExit("unknown op " + op)
        fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print("%-10s %-40s median %8.1f us  min %8.1f us" % (op, os.environ.get("AS_LIB_PATH", "default"),
                                                         float(np.median(ts)), min(ts)))


if __name__ == "__main__":
    main()
