"""Host-side argument handling shared with the reference interface.

Validation rules, the element budget and the seeded core initialisation are
part of the drop-in contract (the GPU run must start from the exact cores the
reference would draw), so they are restated here on the host:
validation.py:8-65, utils.py:9-32, ring.py:62-107.
"""

from __future__ import annotations

import math
import os

import numpy as np

from .errors import ElementBudgetError

DEFAULT_ELEMENT_BUDGET = 1 << 27   # validation.py:8
BUDGET_ENV_VAR = "TENRING_BUDGET"  # validation.py:9


def element_budget(override=None):
    if override is not None:
        return int(override)
    env = os.environ.get(BUDGET_ENV_VAR)
    return int(env) if env is not None else DEFAULT_ELEMENT_BUDGET


def check_element_budget(shape, budget=None):
    limit = element_budget(budget)
    n = math.prod(int(s) for s in shape)
    if n > limit:
        raise ElementBudgetError(
            f"dense tensor with {n} elements exceeds the element budget of "
            f"{limit}; raise it via {BUDGET_ENV_VAR} or an explicit budget")
    return n


def check_dense_tensor(x, min_order=1):
    x = np.asarray(x, dtype=np.float64)
    if x.ndim < min_order:
        raise ValueError(f"tensor order {x.ndim} is below the minimum {min_order}")
    if x.size == 0:
        raise ValueError("tensor has no elements")
    if not np.all(np.isfinite(x)):
        raise ValueError("tensor contains non-finite entries")
    return x


def check_ranks(ranks, order):
    ranks = [int(r) for r in ranks]
    if len(ranks) != order:
        raise ValueError(f"expected {order} ranks, got {len(ranks)}")
    if any(r < 1 for r in ranks):
        raise ValueError("ranks must be positive")
    return ranks


def make_rng(seed=None):
    """Philox4x32 over SeedSequence, exactly as utils.py:9-23."""
    if isinstance(seed, np.random.Generator):
        return seed
    ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    return np.random.Generator(np.random.Philox(ss))


def spawn_seeds(seed, n):
    ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    return ss.spawn(n)


def random_cores(dims, ranks, rng):
    """N(0,1) cores (R_n, I_n, R_{n+1}) drawn in order n = 0..N-1 (ring.py:92-98)."""
    N = len(dims)
    return [rng.standard_normal((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


def zero_cores(dims, ranks):
    N = len(dims)
    return [np.zeros((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


def validate_cores(cores, dims=None):
    cores = [np.asarray(g, dtype=np.float64) for g in cores]
    if len(cores) < 1:
        raise ValueError("a ring needs at least one core")
    for n, g in enumerate(cores):
        if g.ndim != 3:
            raise ValueError(f"core {n} has order {g.ndim}, expected 3")
        nxt = cores[(n + 1) % len(cores)]
        if g.shape[2] != nxt.shape[0]:
            raise ValueError(
                f"bond mismatch between core {n} (right bond {g.shape[2]}) and "
                f"core {(n + 1) % len(cores)} (left bond {nxt.shape[0]})")
    if dims is not None:
        got = tuple(g.shape[1] for g in cores)
        if got != tuple(dims):
            raise ValueError(f"core lateral sizes {got} do not match dims {tuple(dims)}")
    return cores


def core_ranks(cores):
    return tuple(g.shape[0] for g in cores)
