"""Sharded sweeps on the GPU: 2 processes on cuda:0, X split along mode 0 (north_star's "mode 1",
1-based), the real libtrals kernels on every rank, partial right-hand sides all-reduced.

This container's GPU box has one B200, so the two ranks share cuda:0 and talk over gloo (CUDA
tensors staged through the host: no rank's kernels wait on the other's on the device).  The NCCL
path is the same step list with the all-reduces captured in the sweep graph (bench.py checks that
replay against an eager sweep bit for bit on every rank).  Checks: the two replicas end with
bitwise-equal cores and errors, and both equal the single-process run (same public API) to 1e-12.
"""

import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import rel

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

# name: dims, rank_true, noise, seed_data, rank_fit, seed_init, sweeps, variant
CASES = {
    "c3_ne": ((500, 500, 500), 10, 1e-3, 4, 10, 5, 10, "ne"),
    "c3_qr": ((500, 500, 500), 10, 1e-3, 4, 10, 5, 4, "qr"),
    "c5_ne": ((160, 160, 160, 160), 20, 1e-3, 8, 20, 9, 3, "ne"),
    "c2_qrne": ((64, 64, 64, 64), 8, 1e-2, 2, 8, 3, 5, "qrne"),
}


def _data(case):
    from paper_2210_11362_b200.synthetic import SynthSpec, make_dataset
    dims, rt, noise, sd, rf, si, sweeps, variant = CASES[case]
    x, _ = make_dataset(SynthSpec(order=len(dims), dim=dims[0], rank=rt, noise=noise, seed=sd),
                        budget=1 << 40)
    return x


def _run(case, x):
    from paper_2210_11362_b200 import AlsConfig, decompose
    dims, rt, noise, sd, rf, si, sweeps, variant = CASES[case]
    cfg = AlsConfig(ranks=(rf,) * len(dims), max_iters=sweeps, seed=si, error_mode="cheap")
    cores, rep = decompose(x, variant, cfg)
    return cores, list(rep.errors), rep.fallback_count


def _worker(rank, world, port, case, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = _data(case)
    cores, errs, fb = _run(case, x)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), errs=np.array(errs), fb=fb,
             **{f"core_{j}": c for j, c in enumerate(cores)})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("case", sorted(CASES))
def test_two_rank_shard_on_gpu(case, tmp_path):
    # the two ranks share this GPU with the parent: release the parent's cached plans first (the c5
    # engines of the other test modules hold ~20 GB of operand planes each)
    import gc

    import torch
    from paper_2210_11362_b200.solvers import clear_plan_cache
    clear_plan_cache()
    gc.collect()
    torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    port = 29700 + (abs(hash(case)) % 200)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=800)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    r0 = dict(np.load(tmp_path / "rank0.npz"))
    r1 = dict(np.load(tmp_path / "rank1.npz"))
    N = len(CASES[case][0])
    # replicas in lock-step: bitwise
    np.testing.assert_array_equal(r0["errs"], r1["errs"])
    for j in range(N):
        np.testing.assert_array_equal(r0[f"core_{j}"], r1[f"core_{j}"])
    # the same run on one process
    x = _data(case)
    cores, errs, fb = _run(case, x)
    np.testing.assert_allclose(r0["errs"], errs, rtol=0, atol=1e-12)
    assert int(r0["fb"]) == fb
    for j in range(N):
        assert rel(r0[f"core_{j}"], cores[j]) < 1e-12, j
