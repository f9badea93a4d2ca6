"""Generate the BASELINE c5 goldens (160^4, R 20 -> 20, seeds 8 / 9) with the memory-lean oracle.

    python tests/golden/make_c5_golden.py [--variants ne,qrne,qr] [--sweeps 11]

The reference itself cannot run c5 in the 62 GB build container (SURVEY 6:
~65.5 GB peak for NE, more for QR), so the goldens come from `oracle/lean.py`,
the reference's algorithms with the big products blocked (pinned to the
reference's own c2 goldens and the small rings in tests/test_oracle_golden.py).

Output per variant: tests/golden/c5_<variant>.npz with
  x_sum / x_sumsq / x_samples / x_sample_idx  checksums of X (lean.synth)
  exact_errors, cheap_errors                  per sweep, sweeps 1..S
  state<k>_core_<j>                           cores after sweeps k = 5, 6, 10, 11
  fallbacks, seconds                          bookkeeping
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import lean  # noqa: E402
from oracle import tenring_oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
C5 = dict(order=4, dim=160, rank=20, noise=1e-3, seed=8, rank_fit=20, seed_init=9)
KEEP = (5, 6, 10, 11)


def checksums(x):
    flat = x.ravel()
    idx = np.linspace(0, flat.size - 1, 64).astype(np.int64)
    return {"x_sum": float(flat.sum()), "x_sumsq": float(np.dot(flat, flat)), "x_samples": flat[idx],
            "x_sample_idx": idx}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="ne,qrne,qr")
    ap.add_argument("--sweeps", type=int, default=11)
    args = ap.parse_args()
    t0 = time.time()
    x, _ = lean.synth(O.Recipe(order=C5["order"], dim=C5["dim"], rank=C5["rank"], noise=C5["noise"],
                               seed=C5["seed"]))
    cs = checksums(x)
    print(f"synth {time.time() - t0:.1f} s  sum {cs['x_sum']!r} sumsq {cs['x_sumsq']!r}", flush=True)
    dims = (C5["dim"],) * C5["order"]
    ranks = (C5["rank_fit"],) * C5["order"]
    init = O.gaussian_ring(dims, ranks, O.philox(C5["seed_init"]))
    for v in args.variants.split(","):
        t1 = time.time()

        def log(k, run, v=v, t1=t1):
            print(f"{v} sweep {k}: exact {run.exact_errors[-1]!r} cheap {run.cheap_errors[-1]!r} "
                  f"({time.time() - t1:.0f} s)", flush=True)

        run = lean.solve(x, v, ranks, init, args.sweeps, keep=KEEP, log=log)
        rec = dict(cs)
        rec["recipe"] = np.array([C5["order"], C5["dim"], C5["rank"], C5["seed"], C5["rank_fit"], C5["seed_init"],
                                  args.sweeps], dtype=np.int64)
        rec["noise"] = C5["noise"]
        rec["exact_errors"] = np.array(run.exact_errors)
        rec["cheap_errors"] = np.array(run.cheap_errors)
        rec["fallbacks"] = run.fallbacks
        rec["seconds"] = time.time() - t1
        for k, state in run.states.items():
            for j, g in enumerate(state):
                rec[f"state{k}_core_{j}"] = g
        path = os.path.join(OUT, f"c5_{v}.npz")
        np.savez_compressed(path, **rec)
        print(f"wrote {path} ({time.time() - t1:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
