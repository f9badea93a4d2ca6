"""c4 (40^5, R 6 -> 8): model-level distance of our fitted ring to the reference's after 15 sweeps,
per product engine (diagnostic for tests/test_gpu_baseline.py::test_c4_model_level)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import golden_cores, load_golden  # noqa: E402
from oracle import tenring_oracle as O  # noqa: E402
from paper_2210_11362_b200 import AlsConfig, decompose  # noqa: E402

g = load_golden("base_c4")
order, dim, rt, sd, rf, si, sweeps = (int(v) for v in g["recipe"])
x, _ = O.synth(O.Recipe(order=order, dim=dim, rank=rt, noise=float(g["noise"]), seed=sd))
ref = golden_cores(g, "ne_core", order)
b = O.dense_from_ring(ref, budget=1 << 40)
nb = np.linalg.norm(b.ravel())
out = {}
for gemm in ("dmma", "ozaki"):
    for k in (5, 10, 15):
        cores, rep = decompose(x, "ne", AlsConfig(ranks=(rf,) * order, max_iters=k, seed=si, fp64_gemm=gemm))
        if k == 15:
            a = O.dense_from_ring(cores, budget=1 << 40)
            out[f"{gemm}_model15"] = float(np.linalg.norm((a - b).ravel()) / nb)
            out[f"{gemm}_err_maxdiff"] = float(np.max(np.abs(np.array(rep.errors) - g["ne_exact_errors"])))
        out[f"{gemm}_state{k}"] = [c.copy() for c in cores]
# drift between the two engines at sweeps 5 / 10 / 15
for k in (5, 10, 15):
    a = O.dense_from_ring(out[f"dmma_state{k}"], budget=1 << 40)
    c = O.dense_from_ring(out[f"ozaki_state{k}"], budget=1 << 40)
    out[f"engine_drift_model{k}"] = float(np.linalg.norm((a - c).ravel()) / np.linalg.norm(a.ravel()))
print(json.dumps({k: v for k, v in out.items() if "state" not in k}))
