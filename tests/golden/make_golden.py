"""Generate golden vectors by running the REAL reference (`tenring` 0.1.0) in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

The reference tree is not present on the GPU box, so its outputs are frozen
here as .npz fixtures; `tests/test_oracle_golden.py` pins the oracle to them
and the GPU parity tests compare the CUDA path to both.  Inputs too large to
commit (the BASELINE configs' X) are stored as a recipe + checksums: the
oracle's restatement of make_dataset must regenerate the same bytes.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import tenring  # noqa: E402
from tenring import ring, solvers, tensor_ops  # noqa: E402
from tenring.synthetic import SynthSpec, add_noise, make_dataset  # noqa: E402
from tenring.utils import make_rng  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def checksums(x):
    x = np.asarray(x, dtype=np.float64)
    flat = x.ravel()
    idx = np.linspace(0, flat.size - 1, 64).astype(np.int64)
    return {"sum": float(flat.sum()), "sumsq": float(np.dot(flat, flat)), "samples": flat[idx], "sample_idx": idx}


def run_variant(x, variant, ranks, init, sweeps, mode):
    cfg = solvers.AlsConfig(ranks=tuple(ranks), max_iters=sweeps, init_cores=init, error_mode=mode)
    cores, rep = solvers.decompose(x, variant, cfg)
    return cores, rep


def small_cases():
    cases = {}
    # SPEC known answers
    t = np.arange(1, 9, dtype=np.float64).reshape((2, 2, 2), order="F")
    np.savez(os.path.join(OUT, "spec_known.npz"),
             x=t,
             classical_mode1=tensor_ops.classical_unfold(t, 1),
             cyclic_mode1=tensor_ops.cyclic_unfold(t, 1),
             split2=tensor_ops.split_unfold(t, 2))

    def ring_case(name, dims, ranks_true, ranks_fit, noise, seed_data, seed_init, sweeps, variants):
        rng = make_rng(seed_data)
        true = ring.random_cores(dims, ranks_true, rng)
        x = add_noise(ring.reconstruct(true), noise, rng=rng)
        init = ring.random_cores(dims, ranks_fit, make_rng(seed_init))
        rec = {"x": x, "dims": np.array(dims), "ranks": np.array(ranks_fit), "sweeps": sweeps}
        for j, g in enumerate(init):
            rec[f"init_{j}"] = g
        # kernel-level pins from the init cores
        for n in range(len(dims)):
            rec[f"mttsp_{n}"] = tensor_ops.cyclic_unfold(x, n) @ tensor_ops.cyclic_unfold(ring.subchain_skip(init, n), 1)
            rec[f"S_{n}"] = ring.gram_chain(ring.lateral_gram(init[j]) for j in ring.gram_chain_order(n, len(dims)))
        for v in variants:
            for mode in ("exact", "cheap"):
                cores, rep = run_variant(x, v, ranks_fit, init, sweeps, mode)
                rec[f"{v}_{mode}_errors"] = np.array(rep.errors)
                if mode == "exact":
                    for j, g in enumerate(cores):
                        rec[f"{v}_core_{j}"] = g
                rec[f"{v}_{mode}_fallbacks"] = rep.fallback_count
            # per-sweep cores for one-sweep-from-state tests (chained 1-sweep runs == continuous)
            state = init
            for k in range(min(sweeps, 3)):
                state, _ = run_variant(x, v, ranks_fit, state, 1, "none")
                for j, g in enumerate(state):
                    rec[f"{v}_sweep{k + 1}_core_{j}"] = g
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        cases[name] = rec
        print("wrote", name, flush=True)

    # SPEC.md:638 parity protocol shape: N=3, I=30, R=3 (noiseless)
    ring_case("spec_n3_i30_r3", (30, 30, 30), (3, 3, 3), (3, 3, 3), 0.0, 11, 12, 10, ("ne", "qr", "qrne", "als"))
    # non-uniform dims and ranks, N=4, with noise
    ring_case("nonuni_n4", (6, 7, 5, 8), (2, 3, 2, 2), (2, 3, 4, 2), 1e-2, 21, 22, 6, ("ne", "qr", "qrne", "als"))
    # N=5, over-specified rank
    ring_case("n5_i6", (6, 5, 6, 4, 5), (2, 2, 2, 2, 2), (3, 2, 3, 2, 2), 1e-3, 31, 32, 5, ("ne", "qrne"))
    # N=2 edge (matrix)
    ring_case("n2_mat", (20, 30), (3, 3), (3, 2), 1e-2, 41, 42, 6, ("ne", "qr", "qrne", "als"))
    # odd / prime sizes exercise every tail path of the kernels
    ring_case("odd_n3", (13, 7, 11), (2, 3, 2), (3, 2, 3), 1e-2, 51, 52, 5, ("ne", "qr", "als"))
    # rank-deficient blocks: prod_{j != n} I_j < R^2 -> gelsy fallback (NE/QRNE), SVD solve (QR, ALS)
    ring_case("rankdef_n3", (2, 2, 30), (2, 2, 2), (3, 3, 3), 1e-2, 61, 62, 3, ("ne", "qr", "qrne", "als"))
    return cases


def io_and_synth_cases():
    """.dten bytes written by the reference (io.py) and the three synthetic generators (synthetic.py)."""
    from tenring import io as tio
    x = np.arange(60, dtype=np.float64).reshape(3, 4, 5) * 0.5 - 7.25
    x[1, 2, 3] = np.nan
    tio.write_tensor(os.path.join(OUT, "io_3x4x5.dten"), x)
    rec = {}
    specs = {
        "gaussian": SynthSpec(order=3, dim=12, rank=3, kind="gaussian", noise=1e-2, seed=71),
        "congruent": SynthSpec(order=3, dim=12, rank=3, kind="congruent", gamma=0.9, noise=1e-3, seed=72),
        "student_t": SynthSpec(order=4, dim=10, rank=2, kind="student_t", theta=0.7, dof=3, noise=0.0,
                               seed=(7, 3)),
    }
    for kind, spec in specs.items():
        xs, cores = make_dataset(spec)
        rec[f"{kind}_x"] = xs
        for j, g in enumerate(cores):
            rec[f"{kind}_core_{j}"] = g
    np.savez_compressed(os.path.join(OUT, "synth_kinds.npz"), **rec)
    print("wrote io_3x4x5.dten, synth_kinds.npz", flush=True)


def r0_cases():
    """Per-mode R0 of TR-ALS-QR (solvers.py:417-424: mode2_qr of every core, V = subchain_skip of the
    R-tensors, qr_economy of its cyclic 2-unfolding) and of Alg. 1 (solvers.py:337-339: the same with
    the cores themselves), from each small ring's initial cores -- the pins of the GPU R0 merges."""
    from tenring import linalg
    rec = {}
    for name in ("spec_n3_i30_r3", "nonuni_n4", "n5_i6", "n2_mat", "odd_n3", "rankdef_n3"):
        g = np.load(os.path.join(OUT, f"{name}.npz"))
        N = len(g["dims"])
        init = [g[f"init_{j}"] for j in range(N)]
        rts = [ring.mode2_qr(c).r_tensor for c in init]
        for j, r in enumerate(rts):
            rec[f"{name}_rt_{j}"] = r
        for n in range(N):
            _, r0 = linalg.qr_economy(tensor_ops.cyclic_unfold(ring.subchain_skip(rts, n), 1))
            rec[f"{name}_qr_r0_{n}"] = r0
            _, ra = linalg.qr_economy(tensor_ops.cyclic_unfold(ring.subchain_skip(init, n), 1))
            rec[f"{name}_als_r0_{n}"] = ra
    np.savez_compressed(os.path.join(OUT, "r0_modes.npz"), **rec)
    print("wrote r0_modes.npz", flush=True)


BASE_CONFIGS = {
    # name: (order, dim, rank_true, noise, seed_data, rank_fit, seed_init, sweeps, variants)
    "c1": (3, 100, 5, 1e-3, 0, 5, 1, 10, ("ne", "als")),
    "c2": (4, 64, 8, 1e-2, 2, 8, 3, 20, ("ne", "qr")),
    "c3": (3, 500, 10, 1e-3, 4, 10, 5, 10, ("ne", "qr")),
    "c4": (5, 40, 6, 1e-2, 6, 8, 7, 15, ("ne",)),
}


def baseline_config(name, store_cores=True):
    order, dim, rt, noise, sd, rf, si, sweeps, variants = BASE_CONFIGS[name]
    t0 = time.time()
    x, _ = make_dataset(SynthSpec(order=order, dim=dim, rank=rt, kind="gaussian", noise=noise, seed=sd))
    rec = {"recipe": np.array([order, dim, rt, sd, rf, si, sweeps], dtype=np.int64), "noise": noise}
    for k, v in checksums(x).items():
        rec[f"x_{k}"] = v
    init = ring.random_cores([dim] * order, [rf] * order, make_rng(si))
    for v in variants:
        t = time.time()
        cores, rep = run_variant(x, v, [rf] * order, None if False else init, sweeps, "exact")
        rec[f"{v}_exact_errors"] = np.array(rep.errors)
        rec[f"{v}_iter_seconds"] = np.array(rep.iter_seconds)
        if store_cores:
            for j, g in enumerate(cores):
                rec[f"{v}_core_{j}"] = g
        print(name, v, "done in", round(time.time() - t, 1), "s", flush=True)
    # one-sweep-from-state pin for NE: state after sweep 2 -> after sweep 3
    state = init
    for k in range(3):
        prev = state
        state, rep = run_variant(x, "ne", [rf] * order, state, 1, "cheap")
    for j, g in enumerate(prev):
        rec[f"ne_state2_core_{j}"] = g
    for j, g in enumerate(state):
        rec[f"ne_state3_core_{j}"] = g
    rec["ne_state3_cheap_error"] = rep.errors[0]
    np.savez_compressed(os.path.join(OUT, f"base_{name}.npz"), **rec)
    print("wrote", name, "in", round(time.time() - t0, 1), "s", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run the BASELINE configs c1-c4")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    print("tenring", tenring.__version__, "numpy", np.__version__)
    if args.only == "io":
        io_and_synth_cases()
        sys.exit(0)
    if args.only == "r0":
        r0_cases()
        sys.exit(0)
    if args.only is None:
        small_cases()
        io_and_synth_cases()
        r0_cases()
    if args.big or args.only:
        for name in BASE_CONFIGS:
            if args.only and name != args.only:
                continue
            baseline_config(name)
