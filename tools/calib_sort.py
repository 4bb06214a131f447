"""Reference points for the build: CUB-backed torch sorts on the cfg1 key set."""
import numpy as np
import torch

dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
rng = np.random.default_rng(1)
rows = torch.as_tensor(rng.integers(0, 10000, 1_000_000), device=dev)
cols = torch.as_tensor(rng.integers(0, 10000, 1_000_000), device=dev)


def t(fn, reps=10):
    for _ in range(3):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


key64 = cols * 10000 + rows
key32 = key64.to(torch.int32)
print("torch.sort int64 1M (stable)  %.1f us" % t(lambda: torch.sort(key64, stable=True)))
print("torch.sort int32 1M (stable)  %.1f us" % t(lambda: torch.sort(key32, stable=True)))
print("torch.argsort int32 1M        %.1f us" % t(lambda: torch.argsort(key32, stable=True)))
print("coalesce via sparse_coo 1M    %.1f us" % t(lambda: torch.sparse_coo_tensor(torch.stack([rows, cols]), torch.ones(1_000_000, dtype=torch.float64, device=dev), (10000, 10000)).coalesce()))
