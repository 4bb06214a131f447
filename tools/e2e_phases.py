"""Phase times of the build kernel when it reads pinned host triplets
(zero-copy, as bench.py's e2e path does), next to a DMA copy of the same
bytes: is phase 1 running at the copy engine's PCIe rate?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_03380_b200 import SpMat, _kernels, synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
    h = [torch.from_numpy(x).pin_memory() for x in (rows, cols, vals)]
    d = [torch.empty_like(x, device=dev) for x in h]
    for it in range(8):
        m = SpMat.from_triplets(n_rows, n_cols, tuple(h), device=dev).csc()
        torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for it in range(3):
        ev[0].record()
        for x, y in zip(d, h):
            x.copy_(y, non_blocking=True)
        ev[1].record()
        torch.cuda.synchronize()
        print("DMA H2D 24 MB: %.3f ms" % ev[0].elapsed_time(ev[1]), file=sys.stderr)
    for it in range(3):
        ev[0].record()
        m = SpMat.from_triplets(n_rows, n_cols, tuple(h), device=dev).csc()
        ev[1].record()
        torch.cuda.synchronize()
        print("from_triplets (zero-copy in): %.3f ms" % ev[0].elapsed_time(ev[1]), file=sys.stderr)


if __name__ == "__main__":
    main()
