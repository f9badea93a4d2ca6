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


def test_reference_names_exported():
    """Every name of the reference package's surface (pkg/src/tenring/__init__.py:9-37) is importable."""
    import paper_2210_11362_b200 as P
    for name in ("TensorRingALS", "Mode2Qr", "gram_chain", "gram_chain_order", "lateral_gram", "mode2_qr",
                 "random_cores", "reconstruct", "subchain_merge", "subchain_skip", "tr_inner", "tr_norm",
                 "validate_cores", "VARIANTS", "AlsConfig", "AlsReport", "cheap_relative_error", "decompose",
                 "exact_relative_error", "tr_als", "tr_als_ne", "tr_als_qr", "tr_als_qrne", "SynthSpec", "add_noise",
                 "make_dataset", "__version__"):
        assert hasattr(P, name), name
        assert name in P.__all__
    assert P.gram_chain_order(2, 5) == [1, 0, 4, 3]


def test_helpers_have_no_cpu_path():
    """The device helpers fail loudly without a GPU (no silent numpy fallback)."""
    import torch

    import paper_2210_11362_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = np.ones((2, 3, 2))
    with pytest.raises(RuntimeError, match="CUDA"):
        P.lateral_gram(g)
    with pytest.raises(RuntimeError, match="CUDA"):
        P.cheap_relative_error(P.SweepCache(variant="ne", x_norm=1.0, fresh=True, core_mat=np.ones((3, 4)),
                                            m_last=np.ones((3, 4)), s_last=np.eye(4)))
