"""GPU side of the front ends: the .dten reader that lands
X on the device (axis-reversal kernel), make_dataset for every generator kind
vs the reference's own output, the TensorRingALS estimator and the CLI round
trip synth -> decompose against the solver API and the goldens."""

import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden_cores, load_golden, rel
from oracle import tenring_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(7,), (5, 3), (3, 1, 4), (33, 2, 35), (6, 5, 4, 3), (2, 3, 4, 5, 6),
                                  (40, 1, 1, 37), (129, 65)])
def test_reverse_axes_and_read_device(tmp_path, dims):
    from paper_2210_11362_b200 import _lib as L
    from paper_2210_11362_b200.io import read_tensor, read_tensor_device, write_tensor
    rng = np.random.default_rng(len(dims) * 100 + dims[0])
    x = rng.standard_normal(dims)
    p = write_tensor(tmp_path / "x.dten", x)
    got = read_tensor_device(p)
    assert got.is_cuda and got.shape == dims and got.is_contiguous()
    assert np.array_equal(got.cpu().numpy(), read_tensor(p))
    assert np.array_equal(got.cpu().numpy(), x)
    if len(dims) > 1:  # the kernel alone: F-order buffer -> C order
        src = torch.from_numpy(np.ascontiguousarray(x.ravel(order="F"))).cuda()
        dst = torch.empty(dims, dtype=torch.float64, device="cuda")
        L.check(L.lib().trals_reverse_axes_f64(src.data_ptr(), len(dims), L.i64_array(dims), dst.data_ptr(),
                                               int(torch.cuda.current_stream().cuda_stream)), "reverse")
        torch.cuda.synchronize()
        assert np.array_equal(dst.cpu().numpy(), x)


def test_read_device_golden_nan_payload():
    from paper_2210_11362_b200.io import read_tensor_device
    got = read_tensor_device(os.path.join(GOLDEN, "io_3x4x5.dten")).cpu().numpy()
    want = np.arange(60, dtype=np.float64).reshape(3, 4, 5) * 0.5 - 7.25
    want[1, 2, 3] = np.nan
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("kind", ["gaussian", "congruent", "student_t"])
def test_make_dataset_matches_reference(kind):
    from paper_2210_11362_b200.synthetic import SynthSpec, make_dataset
    g = load_golden("synth_kinds")
    spec = {
        "gaussian": SynthSpec(order=3, dim=12, rank=3, kind="gaussian", noise=1e-2, seed=71),
        "congruent": SynthSpec(order=3, dim=12, rank=3, kind="congruent", gamma=0.9, noise=1e-3, seed=72),
        "student_t": SynthSpec(order=4, dim=10, rank=2, kind="student_t", theta=0.7, dof=3, seed=(7, 3)),
    }[kind]
    x, cores = make_dataset(spec)
    assert isinstance(x, np.ndarray) and x.shape == g[f"{kind}_x"].shape
    for a, b in zip(cores, golden_cores(g, f"{kind}_core", spec.order)):
        assert np.array_equal(a, b)
    # GPU reconstruct (half chains + DMMA) vs the reference's CPU subchain: rounding only
    assert rel(x, g[f"{kind}_x"]) < 1e-13
    xd, _ = make_dataset(spec, device="cuda")
    assert xd.is_cuda and rel(xd.cpu().numpy(), g[f"{kind}_x"]) < 1e-13


@pytest.mark.parametrize("variant", ["ne", "qrne"])
def test_estimator_fit_score_reconstruct(variant):
    from paper_2210_11362_b200 import TensorRingALS
    g = load_golden("nonuni_n4")
    dims = tuple(int(d) for d in g["dims"])
    ranks = tuple(int(r) for r in g["ranks"])
    init = golden_cores(g, "init", len(dims))
    est = TensorRingALS(rank=ranks, variant=variant, max_iter=int(g["sweeps"]), error_mode="exact")
    est.fit(g["x"], init_cores=init)
    np.testing.assert_allclose(est.errors_, g[f"{variant}_exact_errors"], rtol=0, atol=1e-9)
    assert est.n_iter_ == int(g["sweeps"]) and est.dims_ == dims
    for j in range(len(dims)):
        assert rel(est.cores_[j], g[f"{variant}_core_{j}"]) < 1e-6
    xh = est.reconstruct()
    ref = O.dense_from_ring(est.cores_)
    assert xh.shape == dims and rel(xh, ref) < 1e-13
    assert abs(est.score(g["x"]) + g[f"{variant}_exact_errors"][-1]) < 1e-9
    with pytest.raises(ValueError, match="fitted on"):
        est.score(np.ones((2, 2)))


def test_cli_synth_then_decompose(tmp_path, capsys):
    from paper_2210_11362_b200 import AlsConfig, decompose
    from paper_2210_11362_b200.cli import main
    from paper_2210_11362_b200.io import read_tensor
    xs = tmp_path / "x.dten"
    assert main(["synth", "--order", "3", "--dim", "16", "--rank", "3", "--kind", "congruent", "--gamma", "0.6",
                 "--noise", "1e-3", "--seed", "4,2", "--out", str(xs), "--truth-cores", str(tmp_path / "truth")]) == 0
    assert "wrote" in capsys.readouterr().out
    assert sorted(os.listdir(tmp_path / "truth")) == ["core_000.dten", "core_001.dten", "core_002.dten"]
    out = tmp_path / "run.json"
    assert main(["decompose", str(xs), "--variant", "ne", "--ranks", "3,3,3", "--max-iters", "6", "--seed", "9",
                 "--error", "exact", "--out", str(out)]) == 0
    rec = json.loads(out.read_text())
    assert rec["variant"] == "ne" and rec["iterations"] == 6 and rec["termination"] == "max_iters"
    assert rec["config"]["dims"] == [16, 16, 16] and len(rec["config"]["cores"]) == 3
    x = read_tensor(xs)
    cores, rep = decompose(x, "ne", AlsConfig(ranks=(3, 3, 3), max_iters=6, seed=9, error_mode="exact"))
    np.testing.assert_allclose(rec["errors"], rep.errors, rtol=0, atol=1e-12)
    for j, pth in enumerate(rec["config"]["cores"]):
        assert rel(read_tensor(pth), cores[j]) < 1e-12
    # the oracle agrees with the CLI run (same seeded init, same X)
    oc, orep = O.solve(x, "ne", O.Config(ranks=(3, 3, 3), max_iters=6, seed=9, error_mode="exact"))
    np.testing.assert_allclose(rec["errors"], orep.errors, rtol=0, atol=1e-9)
