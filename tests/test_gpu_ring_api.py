"""The reference package's ring helpers and cheap-error API (pkg/src/tenring/__init__.py:9-37), on the GPU,
against the oracle (ring.py / solvers.py restatements pinned to the reference)."""

import numpy as np
import pytest

from conftest import rel
from oracle import tenring_oracle as O

pytestmark = pytest.mark.gpu


def _ring(dims, ranks, seed):
    return O.gaussian_ring(dims, ranks, O.philox(seed))


def test_subchain_and_reconstruct():
    import paper_2210_11362_b200 as P
    cores = _ring((5, 6, 4, 3), (2, 3, 2, 4), 1)
    np.testing.assert_allclose(P.subchain_merge(cores[0], cores[1]), O.merge_pair(cores[0], cores[1]),
                               rtol=1e-14, atol=1e-14)
    for n in range(4):
        assert rel(P.subchain_skip(cores, n), O.chain_without(cores, n)) < 1e-14
    assert rel(P.reconstruct(cores), O.dense_from_ring(cores)) < 1e-13
    with pytest.raises(ValueError, match="bond mismatch"):
        P.subchain_merge(cores[0], cores[2][:1])
    with pytest.raises(P.ElementBudgetError):
        P.reconstruct(cores, budget=10)


def test_grams_chain_and_qr():
    import paper_2210_11362_b200 as P
    dims, ranks = (5, 6, 4, 3), (2, 3, 2, 4)
    cores = _ring(dims, ranks, 2)
    for g in cores:
        assert rel(P.lateral_gram(g), O.bond_gram(g)) < 1e-14
    other = _ring(dims, ranks, 3)
    assert rel(P.lateral_gram(cores[1], other[1]), O.bond_gram(cores[1], other[1])) < 1e-14
    for n in range(4):
        assert P.gram_chain_order(n, 4) == O.gram_order(n, 4)
        got = P.gram_chain(P.lateral_gram(cores[j]) for j in P.gram_chain_order(n, 4))
        assert rel(got, O.coefficient_gram(cores, n)) < 1e-13
    for g in cores + [np.random.default_rng(0).standard_normal((3, 20, 2))]:
        f = P.mode2_qr(g)
        o = O.lateral_qr(g)
        assert f.r_tensor.shape == o.r_tensor.shape and f.q.shape == o.q.shape
        assert rel(f.r_tensor, o.r_tensor) < 1e-13 and rel(f.q, o.q) < 1e-13
        np.testing.assert_allclose(f.r_matrix, O.unfold_classical(o.r_tensor, 1), atol=1e-13)


def test_tr_inner_and_norm():
    import paper_2210_11362_b200 as P
    a = _ring((5, 6, 4), (2, 3, 2), 4)
    b = _ring((5, 6, 4), (3, 2, 2), 5)
    want = float(np.vdot(O.dense_from_ring(a), O.dense_from_ring(b)))
    assert abs(P.tr_inner(a, b) - want) <= 1e-12 * abs(want)
    assert abs(P.tr_norm(a) - O.fro(O.dense_from_ring(a))) <= 1e-12 * P.tr_norm(a)
    with pytest.raises(ValueError, match="mode size mismatch"):
        P.tr_inner(a, _ring((5, 6, 3), (2, 3, 2), 6))


@pytest.mark.parametrize("variant", ["ne", "qr", "qrne", "als"])
def test_cheap_relative_error_from_cache(variant):
    """The reference's formula per variant (solvers.py:177-212) from a cache filled from an oracle sweep."""
    import paper_2210_11362_b200 as P
    dims, ranks = (7, 6, 5), (2, 3, 2)
    rng = O.philox(7)
    x = O.noisy(O.dense_from_ring(O.gaussian_ring(dims, ranks, rng)), 1e-2, rng)
    cores, rep = O.solve(x, variant, O.Config(ranks=ranks, max_iters=2, seed=3, error_mode="cheap"))
    # rebuild the last block's intermediates exactly as the oracle's sweep left them
    n = len(dims) - 1
    z = O.unfold_classical(cores[n], 1)
    cache = P.SweepCache(variant=variant, x_norm=O.fro(x), fresh=True, core_mat=z)
    others = [c for c in cores]
    if variant == "ne":
        cache.m_last = O.mttsp(x, others, n)
        cache.s_last = O.coefficient_gram(others, n)
    elif variant == "qrne":
        qrs = [O.lateral_qr(g) for g in others]
        cache.m_last = O.mttsp(x, others, n)
        cache.s_last = O.chain_grams(O.bond_gram(q.r_tensor) for q in (qrs[j] for j in O.gram_order(n, 3)))
        cache.r_core_mat = qrs[n].r_matrix
    elif variant == "qr":
        qrs = [O.lateral_qr(g) for g in others]
        v = O.chain_without([q.r_tensor for q in qrs], n)
        q0, r0 = O.qr_signed(O.unfold_cyclic(v, 1))
        y = O.mode_products(x, [(j, qrs[j].q.T) for j in range(3) if j != n])
        cache.w_last = O.unfold_cyclic(y, n) @ q0
        cache.r0_last = r0
        cache.r_core_mat = qrs[n].r_matrix
    else:
        q, r = O.qr_signed(O.unfold_cyclic(O.chain_without(others, n), 1))
        cache.c_last = q.T @ O.unfold_cyclic(x, n).T
        cache.r_a_last = r
    got = P.cheap_relative_error(cache)
    want = O.residual_exact(x, cores)
    assert abs(got - want) < 1e-9
    cache.fresh = False
    with pytest.raises(P.StaleCacheError):
        P.cheap_relative_error(cache)
