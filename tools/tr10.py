import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1805_03380_b200 import _kernels, synth
n, _, av, ar, ao, B = synth.cfg3_spmm()
dev = torch.device("cuda")
T = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
p, r, v = T(ao, torch.int32), T(ar, torch.int32), T(av, torch.float32)
for _ in range(3):
    _kernels.transpose(n, n, p, r, v)
torch.cuda.synchronize()
