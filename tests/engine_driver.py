"""Drive a SweepEngine directly (test helper): the same call sequence as solvers._run."""

import numpy as np
import torch

from paper_2210_11362_b200.engine import SweepEngine


def run_engine(x, ranks, variant, init_cores, sweeps, lib=None, device="cpu", shard_mode=None, lo=0, hi=None,
               world=1, group=None, exact=False, dtype=np.float64):
    x = np.asarray(x, dtype=dtype)
    dims = x.shape
    if shard_mode is not None and world > 1:
        idx = [slice(None)] * x.ndim
        idx[shard_mode] = slice(lo, hi)
        xl = np.ascontiguousarray(x[tuple(idx)])
    else:
        xl = np.ascontiguousarray(x)
        shard_mode = None
    xt = torch.from_numpy(xl).to(device)
    eng = SweepEngine(xt, dims, ranks, variant, shard_mode=shard_mode, lo=lo, hi=hi, world_size=world, group=group,
                      _test_lib=lib)
    eng.prepare_x()
    eng.compute_xnorm2()
    eng.set_cores(init_cores)
    errs = []
    out = torch.zeros(3, dtype=torch.float64, device=device)
    for _ in range(sweeps):
        eng.run_sweep()
        eng.error_step(out, exact=exact)
        errs.append(float(out[0].item()))
    return eng.cores_host(), errs, eng
