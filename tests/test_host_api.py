"""CPU: the drop-in's argument validation matches the reference (no GPU needed to raise these)."""

import numpy as np
import pytest

from paper_2210_11362_b200 import AlsConfig, ElementBudgetError, decompose, tr_als_ne
from paper_2210_11362_b200.host import make_rng, random_cores
from oracle import tenring_oracle as O


def test_bad_variant_and_modes():
    x = np.ones((3, 3, 3))
    with pytest.raises(ValueError, match="unknown variant"):
        decompose(x, "svd", AlsConfig(ranks=(1, 1, 1)))
    with pytest.raises(ValueError, match="unknown error_mode"):
        tr_als_ne(x, AlsConfig(ranks=(1, 1, 1), error_mode="fast"))
    with pytest.raises(ValueError, match="tol-based"):
        tr_als_ne(x, AlsConfig(ranks=(1, 1, 1), error_mode="none", tol=1e-3))
    with pytest.raises(ValueError, match="max_iters"):
        tr_als_ne(x, AlsConfig(ranks=(1, 1, 1), max_iters=0))


def test_seeded_draws_identical_to_reference_stream():
    dims, ranks = (5, 6, 7), (2, 3, 4)
    a = random_cores(dims, ranks, make_rng(9))
    b = O.gaussian_ring(dims, ranks, O.philox(9))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_budget_guard():
    from paper_2210_11362_b200.host import check_element_budget
    with pytest.raises(ElementBudgetError):
        check_element_budget((1024, 1024, 1024))
    assert check_element_budget((1024, 1024, 1024), budget=1 << 30) == 1 << 30
