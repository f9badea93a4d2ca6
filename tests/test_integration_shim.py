"""INTEGRATION.md's dispatch switch, exercised against the real reference package (build container
only: the reference tree is not on the GPU box).  The GPU solve is replaced by a recorder, so this checks
the wiring -- every front end of the reference (TensorRingALS.fit, the CLI's decompose, tenring.decompose,
the _SOLVERS table) reaches this package's solver with the reference config converted field by field, and
gets the reference's own AlsReport type back -- without a GPU."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")


@pytest.fixture
def tenring(monkeypatch):
    sys.path.insert(0, REF)
    import tenring as t
    from paper_2210_11362_b200 import integration
    from paper_2210_11362_b200 import solvers as ours
    calls = []

    def fake_run(x, config, variant):
        calls.append((np.asarray(x).shape, config, variant))
        dims = np.asarray(x).shape
        ranks = list(config.ranks)
        cores = [np.full((ranks[n], dims[n], ranks[(n + 1) % len(dims)]), 0.5) for n in range(len(dims))]
        rep = ours.AlsReport(variant=variant, errors=[0.25], iter_seconds=[1e-3],
                             iter_buckets=[dict.fromkeys(ours.BUCKETS, 0.0)], termination="max_iters")
        return cores, rep

    monkeypatch.setattr(ours, "_run", fake_run)
    integration.install(t)
    yield t, calls
    integration.uninstall()
    sys.path.remove(REF)


def test_front_ends_dispatch_to_gpu_solvers(tenring, tmp_path):
    t, calls = tenring
    from paper_2210_11362_b200 import solvers as ours
    x = np.random.default_rng(0).standard_normal((4, 5, 6))
    # tenring.decompose and the variant functions
    cores, rep = t.decompose(x, "qr", t.AlsConfig(ranks=(2, 2, 2), max_iters=3, seed=7))
    assert isinstance(rep, t.AlsReport) and rep.errors == [0.25] and rep.variant == "qr"
    assert isinstance(calls[-1][1], ours.AlsConfig) and calls[-1][1].seed == 7 and calls[-1][2] == "qr"
    t.tr_als_ne(x, t.AlsConfig(ranks=(2, 2, 2)))
    assert calls[-1][2] == "ne"
    # the estimator (estimator.py:107)
    est = t.TensorRingALS(rank=2, variant="qrne", max_iter=4, random_state=3).fit(x)
    assert calls[-1][2] == "qrne" and calls[-1][1].max_iters == 4 and est.n_iter_ == 1
    # the CLI (cli.py:65) on a .dten written by the reference's own io
    from tenring import cli, io as tio
    p = tmp_path / "x.dten"
    tio.write_tensor(p, x)
    assert cli.main(["decompose", str(p), "--variant", "ne", "--ranks", "2,2,2", "--out", str(tmp_path / "r.json")]) == 0
    assert calls[-1][2] == "ne" and calls[-1][0] == (4, 5, 6)
    with pytest.raises(ValueError, match="unknown variant"):
        t.decompose(x, "bogus", t.AlsConfig(ranks=(2, 2, 2)))


def test_uninstall_restores_reference():
    sys.path.insert(0, REF)
    try:
        import tenring as t
        from paper_2210_11362_b200 import integration
        before = (t.solvers.decompose, dict(t.solvers._SOLVERS), t.estimator.decompose, t.cli.decompose)
        integration.install(t)
        assert t.solvers.decompose is not before[0]
        integration.uninstall()
        assert (t.solvers.decompose, dict(t.solvers._SOLVERS), t.estimator.decompose, t.cli.decompose) == before
    finally:
        sys.path.remove(REF)
