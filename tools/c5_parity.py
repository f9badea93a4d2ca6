"""One-off full-size BASELINE c5 parity check of a variant against the oracle (GPU box host).

usage: python tools/c5_parity.py [variant] [sweeps]   -> one JSON line with the max deviations.
The oracle is test infrastructure: this script is a checker, not part of the product path.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import tenring_oracle as O  # noqa: E402
from paper_2210_11362_b200 import AlsConfig, decompose  # noqa: E402


def main(variant="qr", sweeps=2):
    order, dim, rt, noise, sd, rf, si = 4, 160, 20, 1e-3, 8, 20, 9
    x, _ = O.synth(O.Recipe(order=order, dim=dim, rank=rt, noise=noise, seed=sd), budget=1 << 40)
    t = time.time()
    cores, rep = decompose(x, variant, AlsConfig(ranks=(rf,) * order, max_iters=sweeps, seed=si, error_mode="cheap"))
    t_gpu = time.time() - t
    t = time.time()
    ocores, orep = O.solve(x, variant, O.Config(ranks=(rf,) * order, max_iters=sweeps, seed=si, error_mode="cheap"))
    t_cpu = time.time() - t
    rel = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(cores, ocores)]
    print(json.dumps({"config": "c5", "variant": variant, "sweeps": sweeps, "errors": list(rep.errors),
                      "oracle_errors": list(orep.errors),
                      "max_err_dev": float(np.max(np.abs(np.array(rep.errors) - np.array(orep.errors)))),
                      "max_core_rel": max(rel), "gpu_call_s": t_gpu, "oracle_s": t_cpu}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "qr", int(sys.argv[2]) if len(sys.argv) > 2 else 2)
