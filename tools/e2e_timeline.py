"""Timeline of one end-to-end build (bench.py's e2e step) split at its
host-visible points: upload (host packing + H2D, until the device has the
triplets), build kernel, the nnz read-back, the D2H of the CSC.  Host
perf_counter marks after a synchronize at each point (so the parts add up to
a slightly slower step than the pipelined one), plus the unsplit step."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import SpMat, _kernels, synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
    n = rows.shape[0]
    h = [torch.from_numpy(x).pin_memory() for x in (rows, cols, vals)]
    o_ptr = torch.empty(n_cols + 1, dtype=torch.int32).pin_memory()
    o_rows = torch.empty(n, dtype=torch.int32).pin_memory()
    o_vals = torch.empty(n, dtype=torch.float64).pin_memory()
    seg = {k: [] for k in ("upload", "build", "nnz_read", "d2h", "split_total", "api_step")}
    for it in range(60):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r, c, v = _kernels.upload_coo(h[0], h[1], h[2], dev, (n_rows, n_cols))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        p, ri, vv, _ = _kernels.coo_to_csc(n_rows, n_cols, r, c, v)  # (reads nnz back inside)
        t2 = time.perf_counter()
        k = ri.shape[0]
        o_ptr.copy_(p, non_blocking=True)
        o_rows[:k].copy_(ri, non_blocking=True)
        o_vals[:k].copy_(vv, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        a0 = time.perf_counter()
        m = SpMat.from_triplets(n_rows, n_cols, tuple(h), device=dev).csc()
        m.to_host(out=(o_ptr, o_rows, o_vals))
        a1 = time.perf_counter()
        if it >= 20:
            seg["upload"].append(t1 - t0)
            seg["build"].append(t2 - t1)
            seg["d2h"].append(t3 - t2)
            seg["split_total"].append(t3 - t0)
            seg["api_step"].append(a1 - a0)
    for k, x in seg.items():
        if x:
            print("%-12s median %7.1f us  min %7.1f us" % (k, 1e6 * statistics.median(x), 1e6 * min(x)))
    # D2H bandwidth alone
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        o_vals.copy_(vv[:n] if vv.shape[0] >= n else torch.zeros(n, dtype=torch.float64, device=dev), non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("D2H 8 MB: %.1f us (%.1f GB/s)" % (1e3 * statistics.median(ts), 8e6 / (statistics.median(ts) * 1e-3) / 1e9))
    ts = []
    hv = h[2]
    dv = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dv.copy_(hv, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("H2D 8 MB: %.1f us (%.1f GB/s)" % (1e3 * statistics.median(ts), 8e6 / (statistics.median(ts) * 1e-3) / 1e9))


if __name__ == "__main__":
    main()
