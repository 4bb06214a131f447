"""Where the time of `.csc()` + the reference-typed host views goes after the
200,000 element writes of cfg 2 (bench.py flush_cfg2_api's csc_ms)."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import SpMat, synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    n_r, n_c, rows, cols, vals = synth.cfg2_writes()
    rl, cl, vl = rows.tolist(), cols.tolist(), vals.tolist()
    seg = {k: [] for k in ("spill", "csc", "to_host", "views", "total")}
    for it in range(8):
        m = SpMat.zeros(n_r, n_c, device=dev)
        for r_, c_, v_ in zip(rl, cl, vl):
            m[r_, c_] = v_
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m._rbt._spill()
        t1 = time.perf_counter()
        d = m.csc()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        p, r, v = d.to_host()
        t3 = time.perf_counter()
        host = (np.asarray(d.values), np.asarray(d.row_indices), np.asarray(d.col_offsets))
        t4 = time.perf_counter()
        if it >= 2:
            for k, a, b in (("spill", t0, t1), ("csc", t1, t2), ("to_host", t2, t3), ("views", t3, t4), ("total", t0, t4)):
                seg[k].append((b - a) * 1e3)
    for k, v in seg.items():
        print("%-8s median %7.3f ms  min %7.3f ms" % (k, statistics.median(v), min(v)))


if __name__ == "__main__":
    main()
