"""Where the end-to-end build time goes: pinned H2D of the int64/f64
triplets, the build, the D2H of the CSC -- CUDA events per segment, plus the
wall time of the public-API call (bench.py's e2e)."""
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
    d = [torch.empty_like(x, device=dev) for x in h]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    seg = {"h2d": [], "build": [], "d2h": [], "api_wall": []}
    o_ptr = torch.empty(n_cols + 1, dtype=torch.int32).pin_memory()
    o_rows = torch.empty(n, dtype=torch.int32).pin_memory()
    o_vals = torch.empty(n, dtype=torch.float64).pin_memory()
    for it in range(25):
        e = [ev() for _ in range(4)]
        e[0].record()
        for x, y in zip(d, h):
            x.copy_(y, non_blocking=True)
        e[1].record()
        p, r, v, _ = _kernels.coo_to_csc(n_rows, n_cols, d[0], d[1], d[2])
        e[2].record()
        k = r.shape[0]
        o_ptr.copy_(p, non_blocking=True)
        o_rows[:k].copy_(r, non_blocking=True)
        o_vals[:k].copy_(v, non_blocking=True)
        e[3].record()
        torch.cuda.synchronize()
        if it >= 5:
            seg["h2d"].append(e[0].elapsed_time(e[1]))
            seg["build"].append(e[1].elapsed_time(e[2]))
            seg["d2h"].append(e[2].elapsed_time(e[3]))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = SpMat.from_triplets(n_rows, n_cols, tuple(h), device=dev).csc()
        kk = m.nnz
        o_ptr.copy_(m.col_ptr, non_blocking=True)
        o_rows[:kk].copy_(m.row_idx, non_blocking=True)
        o_vals[:kk].copy_(m.vals, non_blocking=True)
        torch.cuda.synchronize()
        if it >= 5:
            seg["api_wall"].append((time.perf_counter() - t0) * 1e3)
    for k2, v2 in seg.items():
        print("%-9s median %.3f ms  min %.3f  max %.3f" % (k2, statistics.median(v2), min(v2), max(v2)))
    print("H2D GB/s %.1f, D2H GB/s %.1f" % (24 * n / statistics.median(seg["h2d"]) / 1e6,
                                           (4 * (n_cols + 1) + 12 * k) / statistics.median(seg["d2h"]) / 1e6))


if __name__ == "__main__":
    main()
