"""Both sides of the path on CPU: the .dten format, the
synthetic generators, the run record, the CLI's usage/error contract and the
estimator's sklearn surface -- pinned to files written by the real reference
(tests/golden/make_golden.py: io_3x4x5.dten, synth_kinds.npz)."""

import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, golden_cores, load_golden

from paper_2210_11362_b200 import io as tio
from paper_2210_11362_b200 import synthetic as syn
from paper_2210_11362_b200.host import make_rng, spawn_seeds


def _golden_x():
    x = np.arange(60, dtype=np.float64).reshape(3, 4, 5) * 0.5 - 7.25
    x[1, 2, 3] = np.nan
    return x


def test_write_tensor_bytes_match_reference(tmp_path):
    p = tio.write_tensor(tmp_path / "x.dten", _golden_x())
    assert p.read_bytes() == open(os.path.join(GOLDEN, "io_3x4x5.dten"), "rb").read()


def test_read_tensor_roundtrip_and_nan_payload(tmp_path):
    got = tio.read_tensor(os.path.join(GOLDEN, "io_3x4x5.dten"))
    want = _golden_x()
    assert got.shape == (3, 4, 5) and got.flags["C_CONTIGUOUS"]
    np.testing.assert_array_equal(got, want)  # NaN positions compare equal
    dims, off = tio.read_tensor_header(os.path.join(GOLDEN, "io_3x4x5.dten"))
    assert dims == (3, 4, 5) and off == 12 + 24
    # write -> read is bit exact, NaN payload bits included (io.py:12-13)
    y = np.frombuffer(struct.pack("<Q", 0x7FF8DEADBEEF0001), dtype="<f8").repeat(6).reshape(2, 3)
    p = tio.write_tensor(tmp_path / "y.dten", y)
    assert tio.read_tensor(p).tobytes() == y.tobytes()


@pytest.mark.parametrize("blob,msg", [
    (b"DTE", "truncated header"),
    (b"XTEN" + struct.pack("<II", 1, 1) + struct.pack("<Q", 1) + b"\0" * 8, "bad magic"),
    (b"DTEN" + struct.pack("<II", 2, 1) + struct.pack("<Q", 1) + b"\0" * 8, "unsupported format version 2"),
    (b"DTEN" + struct.pack("<II", 1, 2) + struct.pack("<Q", 1), "truncated dimension list"),
    (b"DTEN" + struct.pack("<II", 1, 0), "truncated dimension list"),
    (b"DTEN" + struct.pack("<II", 1, 2) + struct.pack("<QQ", 2, 0), "nonpositive dimension 0"),
    (b"DTEN" + struct.pack("<II", 1, 1) + struct.pack("<Q", 3) + b"\0" * 16, "payload is 16 bytes, expected 24"),
])
def test_read_tensor_errors_match_reference(tmp_path, blob, msg):
    p = tmp_path / "bad.dten"
    p.write_bytes(blob)
    with pytest.raises(tio.TensorFileError, match=msg):
        tio.read_tensor(p)
    with pytest.raises(tio.TensorFileError, match=msg):
        tio.read_tensor_header(p)


@pytest.mark.parametrize("kind", ["gaussian", "congruent", "student_t"])
def test_generators_bit_identical_to_reference(kind):
    g = load_golden("synth_kinds")
    spec = {
        "gaussian": syn.SynthSpec(order=3, dim=12, rank=3, kind="gaussian", noise=1e-2, seed=71),
        "congruent": syn.SynthSpec(order=3, dim=12, rank=3, kind="congruent", gamma=0.9, noise=1e-3, seed=72),
        "student_t": syn.SynthSpec(order=4, dim=10, rank=2, kind="student_t", theta=0.7, dof=3, seed=(7, 3)),
    }[kind]
    core_seed, _ = spawn_seeds(spec.seed, 2)
    cores = syn._GENERATORS[kind](spec, rng=make_rng(core_seed))
    want = golden_cores(g, f"{kind}_core", spec.order)
    for a, b in zip(cores, want):
        assert a.shape == b.shape and np.array_equal(a, b)


def test_congruent_matrix_gram_and_spec_validation():
    m = syn.congruent_matrix(30, 9, 0.8, make_rng(3))
    G = m.T @ m
    np.testing.assert_allclose(np.diag(G), 1.0, atol=1e-13)
    np.testing.assert_allclose(G[~np.eye(9, dtype=bool)], 0.8, atol=1e-13)
    for bad, msg in [(dict(order=1), "order must be at least 2"), (dict(kind="x"), "unknown core kind"),
                     (dict(noise=-1.0), "noise must be nonnegative"),
                     (dict(kind="congruent", gamma=1.0), "gamma must lie"),
                     (dict(kind="student_t", dof=0), "dof must be at least 1"),
                     (dict(kind="congruent", dim=8, rank=3), "need dim >= rank")]:
        with pytest.raises(ValueError, match=msg):
            syn.SynthSpec(**bad).validate()


def test_run_record_schema():
    from paper_2210_11362_b200 import AlsReport
    rep = AlsReport(variant="ne", errors=[0.5, 0.25], iter_seconds=[0.1, 0.1],
                    iter_buckets=[{"mttsp": 0.05}, {"mttsp": 0.05}], termination="max_iters")
    r = tio.run_record({"input": "x"}, rep, 1.5)
    assert r["schema_version"] == 1 and r["iterations"] == 2 and r["final_error"] == 0.25
    assert set(r) == {"schema_version", "config", "variant", "iterations", "errors", "iter_seconds",
                      "iter_buckets", "upfront_seconds", "termination", "fallback_count", "final_error",
                      "total_seconds", "environment"}
    json.dumps(r)


def test_cli_usage_and_runtime_errors(tmp_path, capsys):
    from paper_2210_11362_b200.cli import main
    with pytest.raises(SystemExit) as e:  # usage error -> 2 (argparse)
        main(["decompose", "x.dten"])
    assert e.value.code == 2
    assert main(["decompose", str(tmp_path / "missing.dten"), "--ranks", "2,2", "--out", str(tmp_path / "r.json")]) == 1
    err = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert err["error"]["type"] == "FileNotFoundError"
    bad = tmp_path / "bad.dten"
    bad.write_bytes(b"XTEN" + b"\0" * 20)
    assert main(["decompose", str(bad), "--ranks", "2,2", "--out", str(tmp_path / "r.json")]) == 1
    err = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert err["error"]["type"] == "TensorFileError" and "bad magic" in err["error"]["message"]
    assert main(["synth", "--order", "1", "--out", str(tmp_path / "s.dten")]) == 1
    err = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert err["error"] == {"type": "ValueError", "message": "order must be at least 2"}


def test_estimator_sklearn_surface():
    from sklearn.base import clone

    from paper_2210_11362_b200 import TensorRingALS
    est = TensorRingALS(rank=(2, 3, 4), variant="ne", max_iter=3, random_state=5)
    p = est.get_params()
    assert p["rank"] == (2, 3, 4) and p["variant"] == "ne" and p["max_iter"] == 3
    c = clone(est).set_params(max_iter=7)
    assert c.max_iter == 7 and est.max_iter == 3
    with pytest.raises(Exception, match="not fitted"):
        est.reconstruct()
    with pytest.raises(ValueError, match="unknown variant"):
        TensorRingALS(variant="bogus").fit(np.ones((3, 3)))
