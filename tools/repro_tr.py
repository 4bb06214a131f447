import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1805_03380_b200 import _kernels
import oracle
n, per, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
rng = np.random.default_rng(3)
R = np.sort(rng.integers(0, n, (n, per)), axis=1)
ok = ~(R[:, 1:] == R[:, :-1]).any(axis=1)
rows = R.reshape(-1); offs = np.arange(0, n * per + 1, per)
vals = rng.standard_normal(n * per)
T = torch.float32 if dt == "f32" else torch.float64
A = (torch.as_tensor(offs.astype(np.int32), device="cuda"), torch.as_tensor(rows.astype(np.int32), device="cuda"), torch.as_tensor(vals, dtype=T, device="cuda"))
out = _kernels.transpose(n, n, *A)
torch.cuda.synchronize()
print("ok", n, per, dt, int(out[0][-1].item()))
