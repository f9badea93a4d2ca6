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


def test_fp64_gemm_option_validated():
    x = np.ones((3, 3, 3))
    with pytest.raises(ValueError, match="unknown fp64_gemm"):
        tr_als_ne(x, AlsConfig(ranks=(1, 1, 1), fp64_gemm="tf32"))


@pytest.mark.parametrize("dims,ranks,want", [((30, 40, 50), (3, 4, 5), "dmma"),      # 2|X|R^2 = 1.5 MFLOP
                                             ((64, 64, 64, 64), (8,) * 4, "dmma"),   # BASELINE c2: 2.1 GFLOP
                                             ((2000, 1100), (32, 32), "ozaki")])     # 4.5 GFLOP
def test_fp64_gemm_auto_policy(dims, ranks, want):
    """fp64_gemm="auto" puts environment products of >= 4 GFLOP (2 |X| R_max^2) on the int8
    tensor cores and leaves the small, launch-bound ones on DMMA; explicit choices stick."""
    import torch
    from fake_trals import FakeTrals
    from paper_2210_11362_b200.engine import OZ64_MIN_FLOPS, SweepEngine
    x = torch.zeros(dims, dtype=torch.float64)
    assert (2.0 * x.numel() * max(ranks) ** 2 >= OZ64_MIN_FLOPS) == (want == "ozaki")
    assert SweepEngine(x, dims, ranks, "ne", _test_lib=FakeTrals()).fp64_gemm == want
    assert SweepEngine(x, dims, ranks, "ne", fp64_gemm="dmma", _test_lib=FakeTrals()).fp64_gemm == "dmma"
    with pytest.raises(ValueError, match="unknown fp64_gemm"):
        SweepEngine(x, dims, ranks, "ne", fp64_gemm="fast", _test_lib=FakeTrals())
