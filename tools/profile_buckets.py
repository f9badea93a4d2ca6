"""Per-bucket device time of a sweep (CUDA events at bucket boundaries) for the BASELINE configs."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200 import AlsConfig, decompose  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402

for name in sys.argv[1:] or ["c2", "c5"]:
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
    x, _ = make_dataset_device(order, dim, rt, noise, sd)
    for variant in ("ne",):
        cfg = AlsConfig(ranks=(rf,) * order, max_iters=5, seed=si, error_mode="cheap")
        decompose(x, variant, cfg)
        cores, rep = decompose(x, variant, cfg)
        b = {k: float(np.mean([d[k] for d in rep.iter_buckets[1:]])) * 1e3 for k in rep.iter_buckets[0]}
        print(json.dumps({"config": name, "variant": variant, "sweep_ms": float(np.mean(rep.iter_seconds[1:])) * 1e3,
                          "bucket_ms": b}))
    del x
    torch.cuda.empty_cache()
