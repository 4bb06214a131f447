import os, sys, time, statistics
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1805_03380_b200 import SpMat, synth
from paper_1805_03380_b200 import csc as C
from paper_1805_03380_b200.csc import Dims
dev = torch.device("cuda")
n_rows, n_cols, rows, cols, vals = synth.cfg1_triplets()
n = rows.shape[0]
h = [torch.from_numpy(x).pin_memory() for x in (rows, cols, vals)]
o = (torch.empty(n_cols + 1, dtype=torch.int32).pin_memory(), torch.empty(n, dtype=torch.int32).pin_memory(),
     torch.empty(n, dtype=torch.float64).pin_memory())
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
sc = torch.empty((), dtype=torch.int64, device=dev)
def spmat():
    m = SpMat.from_triplets(n_rows, n_cols, tuple(h), device=dev).csc()
    k = m.nnz
    o[0].copy_(m.col_ptr, non_blocking=True); o[1][:k].copy_(m.row_idx, non_blocking=True); o[2][:k].copy_(m.vals, non_blocking=True)
def host():
    C.canonicalize_host(Dims(n_rows, n_cols), *h, out=o)
def run(fn, name, flush_on):
    ts = []
    for i in range(40):
        if flush_on: torch.sum(flush.view(torch.int64), dim=0, out=sc)
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, "flush" if flush_on else "noflush", round(statistics.median(ts[10:]) * 1e3, 3))
for fl in (True, False):
    run(spmat, "spmat", fl); run(host, "host", fl); run(spmat, "spmat", fl); run(host, "host", fl)
