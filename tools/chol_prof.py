"""Time (CUDA events) or profile the m x m SPD factorisation + solve used per mode (trals_cholesky_f64 /
trals_chol_solve_f64).  usage: python tools/chol_prof.py [m=400] [rows=160] [reps=20]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import device_ops as ops  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 400
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 160
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rng = np.random.default_rng(0)
a = rng.standard_normal((2 * m, m))
S = torch.from_numpy(a.T @ a).cuda()
M = torch.from_numpy(rng.standard_normal((rows, m))).cuda()
f = ops.cholesky(S)
z = ops.chol_solve(f, M)
torch.cuda.synchronize()
print("residual", float((z @ S - M).norm() / M.norm()), "info", f.info.tolist())
for name, fn in (("cholesky", lambda: ops.cholesky(S)), ("solve", lambda: ops.chol_solve(f, M))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} m={m}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us")
