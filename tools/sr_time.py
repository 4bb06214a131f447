"""Event-timed build / transpose / flush on their BASELINE configs through the
raw C ABI (L2 flushed before every rep), with optional per-phase timestamps:
    AS_PHASE_TIMES=1 python tools/sr_time.py [build transpose flush] [reps]
Prints median / min event time per op (us)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1805_03380_b200 import _lib, synth  # noqa: E402
from paper_1805_03380_b200._lib import ptr  # noqa: E402


def main():
    args = [x for x in sys.argv[1:] if x != "--noflush"]
    noflush = "--noflush" in sys.argv
    reps = int(args[-1]) if args and args[-1].isdigit() else 20
    ops = [a for a in args if not a.isdigit()] or ["build", "transpose", "flush"]
    dev = torch.device("cuda")
    L = _lib.lib()
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    scratch = torch.empty((), dtype=torch.int64, device=dev)

    def T(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            if not noflush:
                torch.sum(flush.view(torch.int64), dim=0, out=scratch)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts), min(ts)

    n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
    for op in ops:
        if op == "build":
            n = rows.shape[0]
            r, c, v = T(rows, torch.int32), T(cols, torch.int32), T(vals, torch.float64)
            cp = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
            ri = torch.empty(n, dtype=torch.int32, device=dev)
            ov = torch.empty(n, dtype=torch.float64, device=dev)
            info = torch.empty(2, dtype=torch.int64, device=dev)
            wb = L.as_build_workspace_bytes(n, n_cols)
            ws = torch.empty(wb, dtype=torch.uint8, device=dev)
            fn = lambda: _lib.check(L.as_coo_to_csc_f64(n_rows, n_cols, n, ptr(r), ptr(c), 4, ptr(v), 0, ptr(cp),
                                                         ptr(ri), ptr(ov), ptr(info), ptr(ws), wb, sp))
        elif op == "transpose":
            A = oracle.canonicalize(n_rows, n_cols, rows, cols, vals)
            p, r, v = T(A[2], torch.int32), T(A[1], torch.int32), T(A[0], torch.float64)
            nnz = int(r.shape[0])
            tp = torch.empty(n_rows + 1, dtype=torch.int32, device=dev)
            tr = torch.empty(nnz, dtype=torch.int32, device=dev)
            tv = torch.empty(nnz, dtype=torch.float64, device=dev)
            wb = L.as_transpose_workspace_bytes(nnz, n_rows)
            ws = torch.empty(wb, dtype=torch.uint8, device=dev)
            fn = lambda: _lib.check(L.as_csc_transpose_f64(n_rows, n_cols, nnz, ptr(p), ptr(r), ptr(v), ptr(tp),
                                                            ptr(tr), ptr(tv), ptr(ws), wb, sp))
        elif op == "flush":
            n2, _, r2, c2, v2 = synth.cfg2_writes()
            nl = r2.shape[0]
            lr, lc, lv = T(r2, torch.int32), T(c2, torch.int32), T(v2, torch.float64)
            bp = torch.zeros(n2 + 1, dtype=torch.int32, device=dev)
            br = torch.empty(0, dtype=torch.int32, device=dev)
            bv = torch.empty(0, dtype=torch.float64, device=dev)
            op_ = torch.empty(n2 + 1, dtype=torch.int32, device=dev)
            orr = torch.empty(nl, dtype=torch.int32, device=dev)
            ov2 = torch.empty(nl, dtype=torch.float64, device=dev)
            info = torch.empty(2, dtype=torch.int64, device=dev)
            wb = L.as_flush_workspace_bytes(0, nl, n2)
            ws = torch.empty(wb, dtype=torch.uint8, device=dev)
            fn = lambda: _lib.check(L.as_flush_log_f64(n2, n2, 0, ptr(bp), ptr(br), ptr(bv), nl, ptr(lr), ptr(lc),
                                                        ptr(lv), ptr(op_), ptr(orr), ptr(ov2), ptr(info), ptr(ws), wb,
                                                        sp))
        elif op == "empty":
            z = torch.empty(1, dtype=torch.int32, device=dev)
            fn = lambda: z.zero_()
        else:
            raise SystemExit("unknown op " + op)
        med, mn = timeit(fn)
        print("%-10s median %8.2f us  min %8.2f us" % (op, med, mn), flush=True)


if __name__ == "__main__":
    main()
