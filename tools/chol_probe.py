"""ncu fodder: the resident Cholesky+inverse kernel at m = 64 (c2/c4 size)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import ops  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rng = np.random.default_rng(m)
a = rng.standard_normal((2 * m, m))
s = torch.from_numpy(a.T @ a).cuda()
for _ in range(3):
    f = ops.cholesky(s)
torch.cuda.synchronize()
print("ok")
