"""The oracle (oracle/tenring_oracle.py) pinned to vectors produced by the real reference.

CPU only.  Fixtures: tests/golden/*.npz from tests/golden/make_golden.py.
"""

import numpy as np
import pytest

from conftest import golden_cores, load_golden, rel
from oracle import tenring_oracle as O

SMALL = ["spec_n3_i30_r3", "nonuni_n4", "n5_i6", "n2_mat", "odd_n3", "rankdef_n3"]


def test_spec_known_answers():
    g = load_golden("spec_known")
    t = g["x"]
    # SPEC.md:48 / :58 / :68 -- classical, cyclic and split unfoldings of the 2x2x2 tensor 1..8
    assert np.array_equal(O.unfold_classical(t, 1), g["classical_mode1"])
    assert np.array_equal(O.unfold_classical(t, 1), np.array([[1, 2, 5, 6], [3, 4, 7, 8]], dtype=float))
    assert np.array_equal(O.unfold_cyclic(t, 1), g["cyclic_mode1"])
    assert np.array_equal(O.unfold_cyclic(t, 1), np.array([[1, 5, 2, 6], [3, 7, 4, 8]], dtype=float))
    assert np.array_equal(O.unfold_split(t, 2), g["split2"])


def test_tri_solve_known_answer():
    # z @ r.T = rhs with r = [[2,1],[0,1]], rhs = [[1,1]] -> [[0,1]]
    z = O.solve_upper_right(np.array([[2.0, 1.0], [0.0, 1.0]]), np.array([[1.0, 1.0]]))
    assert np.allclose(z, [[0.0, 1.0]])


@pytest.mark.parametrize("name", SMALL)
def test_kernel_level_pins(name):
    g = load_golden(name)
    dims = tuple(int(d) for d in g["dims"])
    N = len(dims)
    init = golden_cores(g, "init", N)
    for n in range(N):
        assert rel(O.mttsp(g["x"], init, n), g[f"mttsp_{n}"]) < 1e-13
        assert rel(O.coefficient_gram(init, n), g[f"S_{n}"]) < 1e-13


@pytest.mark.parametrize("name", SMALL)
def test_solver_pins(name):
    g = load_golden(name)
    dims = tuple(int(d) for d in g["dims"])
    N = len(dims)
    ranks = tuple(int(r) for r in g["ranks"])
    init = golden_cores(g, "init", N)
    sweeps = int(g["sweeps"])
    for v in ("ne", "qr", "qrne", "als"):
        if f"{v}_exact_errors" not in g:
            continue
        for mode in ("exact", "cheap"):
            cores, rep = O.solve(g["x"], v, O.Config(ranks=ranks, max_iters=sweeps, init_cores=init, error_mode=mode))
            assert np.max(np.abs(np.array(rep.errors) - g[f"{v}_{mode}_errors"])) < 1e-12
            assert rep.fallback_count == int(g[f"{v}_{mode}_fallbacks"])
            if mode == "exact":
                for j in range(N):
                    assert rel(cores[j], g[f"{v}_core_{j}"]) < 1e-10


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_baseline_recipe_regenerates_x(name):
    """The oracle's make_dataset restatement reproduces the reference's X (checksums + samples)."""
    g = load_golden(f"base_{name}")
    order, dim, rt, sd, rf, si, sweeps = (int(v) for v in g["recipe"])
    if dim ** order > 20_000_000:
        pytest.skip("large config regenerated only in the slow suite")
    x, _ = O.synth(O.Recipe(order=order, dim=dim, rank=rt, noise=float(g["noise"]), seed=sd))
    flat = x.ravel()
    assert abs(flat.sum() - g["x_sum"]) <= 1e-9 * abs(g["x_sumsq"]) ** 0.5 * flat.size ** 0.5
    assert abs(np.dot(flat, flat) - g["x_sumsq"]) <= 1e-12 * g["x_sumsq"]
    assert np.allclose(flat[g["x_sample_idx"]], g["x_samples"], rtol=1e-12, atol=0)


def test_c1_oracle_matches_reference_run():
    g = load_golden("base_c1")
    order, dim, rt, sd, rf, si, sweeps = (int(v) for v in g["recipe"])
    x, _ = O.synth(O.Recipe(order=order, dim=dim, rank=rt, noise=float(g["noise"]), seed=sd))
    cores, rep = O.solve(x, "ne", O.Config(ranks=(rf,) * order, max_iters=sweeps, seed=si))
    assert np.max(np.abs(np.array(rep.errors) - g["ne_exact_errors"])) < 1e-12
    for j in range(order):
        assert rel(cores[j], g[f"ne_core_{j}"]) < 1e-10
