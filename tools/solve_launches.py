"""Launch list fodder: blocked Cholesky + solve at m=400, rows=160 (c5 sizes)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import ops  # noqa: E402

m, rows = int(sys.argv[1]) if len(sys.argv) > 1 else 400, 160
rng = np.random.default_rng(0)
a = rng.standard_normal((2 * m, m))
s = torch.from_numpy(a.T @ a).cuda()
M = torch.from_numpy(rng.standard_normal((rows, m))).cuda()
for _ in range(3):
    f = ops.cholesky(s)
    z = ops.chol_solve(f, M)
torch.cuda.synchronize()
print("ok", float(z.abs().sum()))
