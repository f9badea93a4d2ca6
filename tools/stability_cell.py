"""SPEC acceptance criterion 8 (paper Fig. 4, desk scale): experiment B-II cell
eta = 1e-10, gamma = 1 - 1e-10 on a 100^3 rank-5 congruent tensor -- per-trial final
exact errors of NE / QR / QRNE (the reference's bench seeding: data (seed,0,tag,trial),
init (seed,1,tag,trial)).

    python tools/stability_cell.py [trials] [gap] [eta]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_11362_b200 import AlsConfig, decompose  # noqa: E402
from paper_2210_11362_b200.synthetic import SynthSpec, make_dataset  # noqa: E402


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    gap = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
    eta = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-10
    res = {v: [] for v in ("ne", "qr", "qrne")}
    for trial in range(trials):
        spec = SynthSpec(order=3, dim=100, rank=5, kind="congruent", noise=eta, gamma=1 - gap, seed=(0, 0, 0, trial))
        x, _ = make_dataset(spec, device="cuda")
        for v in res:
            _, rep = decompose(x, v, AlsConfig(ranks=[5] * 3, max_iters=20, seed=(0, 1, 0, trial),
                                               error_mode="exact", timing_buckets=False))
            res[v].append(rep.errors[-1])
    out = {v: {"median": float(np.median(e)), "errors": [float(t) for t in e]} for v, e in res.items()}
    out["qr_beats_ne"] = int(sum(a < b for a, b in zip(res["qr"], res["ne"])))
    out["qrne_beats_ne"] = int(sum(a < b for a, b in zip(res["qrne"], res["ne"])))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
