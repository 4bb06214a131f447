"""Calibrate event-timed device throughput with plain torch ops (HBM-cold)."""
import torch

dev = torch.device("cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
scratch = torch.empty(1, dtype=torch.int64, device=dev)


def t(fn, reps=10):
    for _ in range(3):
        torch.sum(flush.view(torch.int64), dim=0, out=scratch)
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.sum(flush.view(torch.int64), dim=0, out=scratch)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for n in (1 << 18, 1 << 20, 10 << 20, 50 << 20):
    x = torch.ones(n, dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    us_sum = t(lambda: x.sum())
    us_copy = t(lambda: y.copy_(x))
    print("int32 n=%9d  sum %8.2f us (%6.0f GB/s)  copy %8.2f us (%6.0f GB/s)" % (
        n, us_sum, 4 * n / us_sum / 1e3, us_copy, 8 * n / us_copy / 1e3))
print("empty kernel", t(lambda: scratch.zero_()))
