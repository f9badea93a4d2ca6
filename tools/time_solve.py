"""Device time of the small dense kernels (Cholesky, row-parallel solve, Gram chain) at the BASELINE sizes."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import ops  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


for m, rows in [(25, 100), (64, 64), (100, 500), (64, 40), (400, 160)]:
    rng = np.random.default_rng(m)
    a = rng.standard_normal((2 * m, m))
    s = torch.from_numpy(a.T @ a).cuda()
    M = torch.from_numpy(rng.standard_normal((rows, m))).cuda()
    f = ops.cholesky(s)
    t_chol = timeit(lambda: ops.cholesky(s))
    t_solve = timeit(lambda: ops.chol_solve(f, M))
    print(json.dumps({"m": m, "rows": rows, "cholesky_us": round(t_chol, 1), "chol_solve_us": round(t_solve, 1)}))
