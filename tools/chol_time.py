"""Time the blocked Cholesky at m = 400 (c5's R^2) and list its launches under ncu."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import ops  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 400
rng = np.random.default_rng(0)
a = rng.standard_normal((3 * m, m))
s = torch.tensor(a.T @ a, device="cuda")
for _ in range(3):
    ops.cholesky(s)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.cholesky(s)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1000)
ts.sort()
print(f"cholesky m={m}: median {ts[len(ts) // 2]:.1f} us")
