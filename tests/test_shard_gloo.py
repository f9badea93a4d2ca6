"""Sharded sweep (X split along one mode, partial M_n all-reduced) on 2 CPU ranks over gloo.

Runs the engine's real multi-rank step list (torch.distributed.all_reduce on
the partial right-hand sides, local core rows for the sharded mode, zero-
padded M_s) through the numpy C-ABI model and checks every rank ends with
cores identical to each other and equal to the single-process oracle.
"""

import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _worker(rank, world, port, case, out_q):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist
    from engine_driver import run_engine
    from fake_trals import FakeTrals
    from oracle import tenring_oracle as O
    from paper_2210_11362_b200.solvers import _slab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dims, ranks, shard, variant, exact = case
    rng = np.random.default_rng(7)
    x = rng.standard_normal(dims)
    init = O.gaussian_ring(dims, ranks, O.philox(3))
    lo, hi = _slab(dims[shard], world, rank)
    cores, errs, _ = run_engine(x, list(ranks), variant, init, 2, lib=FakeTrals(), shard_mode=shard, lo=lo, hi=hi,
                                world=world, exact=exact)
    out_q.put((rank, [c.tolist() for c in cores], errs))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    ((7, 9, 5), (2, 3, 2), 1, "ne", False),
    ((5, 4, 6, 3), (2, 3, 2, 2), 1, "ne", False),
    ((5, 4, 6, 3), (2, 3, 2, 2), 3, "ne", False),
    ((6, 5, 4, 3, 4), (2, 2, 2, 2, 2), 0, "ne", False),
    ((5, 4, 6, 3), (2, 3, 2, 2), 0, "qr", False),      # per-core QR + R-Gram chain on every rank
    ((7, 9, 5), (2, 3, 2), 2, "qrne", True),           # exact error: partial residuals all-reduced
    ((6, 5, 4, 3, 4), (2, 2, 2, 2, 2), 4, "qrne", False),
])
def test_two_rank_shard_matches_oracle(case):
    from oracle import tenring_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (abs(hash(str(case))) % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, cores, errs = q.get(timeout=120)
        res[r] = (cores, errs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dims, ranks, shard, variant, exact = case
    rng = np.random.default_rng(7)
    x = rng.standard_normal(dims)
    init = O.gaussian_ring(dims, ranks, O.philox(3))
    ocores, rep = O.solve(x, variant, O.Config(ranks=ranks, max_iters=2, init_cores=init,
                                               error_mode="exact" if exact else "cheap"))
    c0, e0 = res[0]
    c1, e1 = res[1]
    assert e0 == e1  # replicas stay in lock-step
    np.testing.assert_allclose(e0, rep.errors, rtol=0, atol=1e-12)
    for j in range(len(dims)):
        np.testing.assert_array_equal(np.array(c0[j]), np.array(c1[j]))
        np.testing.assert_allclose(np.array(c0[j]), ocores[j], rtol=1e-9, atol=1e-9)
