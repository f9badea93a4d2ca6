"""Fallback counts of the BASELINE configs (is the pinv/gelsy path firing?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200 import AlsConfig, decompose  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
    x, _ = make_dataset_device(order, dim, rt, noise, sd)
    for v in ("ne", "qr"):
        _, rep = decompose(x, v, AlsConfig(ranks=(rf,) * order, max_iters=sweeps, seed=si, error_mode="cheap"))
        print(name, v, "fallbacks", rep.fallback_count, "final", rep.errors[-1], flush=True)
    del x
