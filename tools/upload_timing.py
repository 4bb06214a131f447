"""Timing of the narrowing upload (as_upload_coo_i64) against plain copies:
host wall time of the call, device time of its copies, and the whole
from_triplets + read-back step."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import _kernels, synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
    h = [torch.from_numpy(x).pin_memory() for x in (rows, cols, vals)]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    res = {"call_wall": [], "dev_total": [], "plain_h2d24": [], "plain_h2d16": []}
    d = [torch.empty_like(x, device=dev) for x in h]
    h32 = [torch.empty(x.shape[0], dtype=torch.int32).pin_memory() for x in h[:2]]
    d32 = [torch.empty(x.shape[0], dtype=torch.int32, device=dev) for x in h[:2]]
    for it in range(30):
        torch.cuda.synchronize()
        ev[0].record()
        t0 = time.perf_counter()
        _kernels.upload_coo(h[0], h[1], h[2], dev)
        t1 = time.perf_counter()
        ev[1].record()
        torch.cuda.synchronize()
        if it >= 5:
            res["call_wall"].append((t1 - t0) * 1e3)
            res["dev_total"].append(ev[0].elapsed_time(ev[1]))
        ev[0].record()
        for x, y in zip(d, h):
            x.copy_(y, non_blocking=True)
        ev[1].record()
        for x, y in zip(d32, h32):
            x.copy_(y, non_blocking=True)
        d[2].copy_(h[2], non_blocking=True)
        ev[2].record()
        torch.cuda.synchronize()
        if it >= 5:
            res["plain_h2d24"].append(ev[0].elapsed_time(ev[1]))
            res["plain_h2d16"].append(ev[1].elapsed_time(ev[2]))
    for k, v in res.items():
        print("%-12s median %.3f ms  min %.3f" % (k, statistics.median(v), min(v)))


if __name__ == "__main__":
    main()
