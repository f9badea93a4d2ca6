"""Synthetic TR tensors generated on the GPU (the §8(f) "GPU-side reconstruct" row).

Same recipes as the reference (pkg/src/tenring/synthetic.py): `SynthSpec`
(:40-81), the gaussian / congruent / student_t core generators (:84-151), the
relative-noise model (:167-181) and `make_dataset` (:184-197).  The true cores
are drawn on the host with the reference's Philox streams, in the same order and
with the same calls, so they are bit-identical; the dense tensor is then
reconstructed on the device with libtrals (two half chains + one DMMA GEMM,
instead of the reference's full subchain materialisation, ring.py:155-170).
`make_dataset` keeps the reference's host noise stream (identical output up to
reconstruct rounding); `make_dataset_device` (the bench's) draws the noise on
the device instead.
"""

from __future__ import annotations

import numpy as np
import torch

from dataclasses import dataclass

from . import _lib as L
from .host import check_element_budget, make_rng, spawn_seeds

CORE_KINDS = ("gaussian", "congruent", "student_t")   # synthetic.py:37


@dataclass
class SynthSpec:
    """One synthetic tensor recipe (synthetic.py:40-81): `order` cubic modes of
    size `dim`, true bond dimension `rank`, core generator `kind`, relative
    `noise`; `gamma` (congruent), `theta` / `dof` (student_t); `seed` int/tuple."""

    order: int = 3
    dim: int = 100
    rank: int = 5
    kind: str = "gaussian"
    noise: float = 0.0
    gamma: float = 0.5
    theta: float = 0.5
    dof: int = 1
    seed: object = None

    def validate(self):
        if self.order < 2:
            raise ValueError("order must be at least 2")
        if self.dim < 1 or self.rank < 1:
            raise ValueError("dim and rank must be positive")
        if self.kind not in CORE_KINDS:
            raise ValueError(f"unknown core kind {self.kind!r}; expected {CORE_KINDS}")
        if self.noise < 0:
            raise ValueError("noise must be nonnegative")
        if self.kind == "congruent" and not 0.0 <= self.gamma < 1.0:
            raise ValueError("gamma must lie in [0, 1)")
        if self.kind == "student_t":
            if not 0.0 <= self.theta < 1.0:
                raise ValueError("theta must lie in [0, 1)")
            if self.dof < 1:
                raise ValueError("dof must be at least 1")
        if self.kind in ("congruent", "student_t") and self.dim < self.rank ** 2:
            raise ValueError(f"matrix-based cores need dim >= rank^2 ({self.dim} < {self.rank ** 2})")
        return self


def _signed_qr_q(a):
    """Q of the economy QR with a nonnegative R diagonal (linalg.py:36-52)."""
    q, r = np.linalg.qr(np.asarray(a, dtype=np.float64), mode="reduced")
    d = np.sign(np.diagonal(r)).copy()
    d[d == 0] = 1.0
    return q * d


def _core_from_matrix(m, rank):
    """(I x R^2) matrix -> (R, I, R) core: m is the core's classical mode-1
    unfolding, column = left bond + R * right bond (synthetic.py:8-10, tensor_ops.py:100-108)."""
    dim = m.shape[0]
    return np.ascontiguousarray(np.asarray(m).reshape(dim, rank, rank, order="F").transpose(1, 0, 2))


def gaussian_cores(spec, rng=None):
    """N(0, 1) cores (rank, dim, rank), drawn in mode order (synthetic.py:84-91)."""
    spec.validate()
    rng = rng if rng is not None else make_rng(spec.seed)
    return [rng.standard_normal((spec.rank, spec.dim, spec.rank)) for _ in range(spec.order)]


def congruent_matrix(rows, cols, gamma, rng):
    """Unit-norm columns with every pairwise inner product equal to `gamma`
    (synthetic.py:94-111): Q (orthonormal, from a Gaussian draw) times the
    symmetric square root a I + b J of (1 - gamma) I + gamma J."""
    if not 0.0 <= gamma < 1.0:
        raise ValueError("gamma must lie in [0, 1)")
    if rows < cols:
        raise ValueError(f"need rows >= cols for orthonormal columns ({rows} < {cols})")
    q = _signed_qr_q(rng.standard_normal((rows, cols)))
    a = np.sqrt(1.0 - gamma)
    b = (np.sqrt(1.0 - gamma + cols * gamma) - a) / cols
    return q @ (a * np.eye(cols) + b * np.ones((cols, cols)))


def congruent_cores(spec, rng=None):
    """Cores from congruence-gamma (dim x rank^2) matrices (synthetic.py:118-130)."""
    spec.validate()
    if spec.kind != "congruent":
        raise ValueError(f"spec kind is {spec.kind!r}, expected 'congruent'")
    rng = rng if rng is not None else make_rng(spec.seed)
    return [_core_from_matrix(congruent_matrix(spec.dim, spec.rank ** 2, spec.gamma, rng), spec.rank)
            for _ in range(spec.order)]


def student_t_matrix(rows, cols, theta, dof, rng):
    """Rows of multivariate-t draws, correlation theta^|i-j|, `dof` degrees of freedom
    (synthetic.py:133-147): a correlated Gaussian row over sqrt(chi2_dof / dof)."""
    if not 0.0 <= theta < 1.0:
        raise ValueError("theta must lie in [0, 1)")
    lag = np.abs(np.subtract.outer(np.arange(cols), np.arange(cols)))
    lower = np.linalg.cholesky(theta ** lag)
    g = rng.standard_normal((rows, cols)) @ lower.T
    return g / np.sqrt(rng.chisquare(dof, size=rows) / dof)[:, None]


def student_t_cores(spec, rng=None):
    """Cores from correlated multivariate-t (dim x rank^2) matrices (synthetic.py:150-161)."""
    spec.validate()
    if spec.kind != "student_t":
        raise ValueError(f"spec kind is {spec.kind!r}, expected 'student_t'")
    rng = rng if rng is not None else make_rng(spec.seed)
    return [_core_from_matrix(student_t_matrix(spec.dim, spec.rank ** 2, spec.theta, spec.dof, rng), spec.rank)
            for _ in range(spec.order)]


_GENERATORS = {"gaussian": gaussian_cores, "congruent": congruent_cores, "student_t": student_t_cores}


def add_noise(x_true, eta, seed=None, rng=None):
    """x + eta * (||x|| / ||n||) * n with n ~ N(0, 1) from the reference stream
    (synthetic.py:167-181); x_true may be a host array or a CUDA tensor (then the
    draw is uploaded and the update runs on the device)."""
    if eta < 0:
        raise ValueError("eta must be nonnegative")
    if eta == 0.0:
        return x_true
    rng = rng if rng is not None else make_rng(seed)
    draw = rng.standard_normal(tuple(x_true.shape))
    dn = float(np.linalg.norm(draw.ravel()))
    if isinstance(x_true, torch.Tensor):
        d = torch.from_numpy(draw).to(x_true.device)
        return x_true + (eta * float(_sumsq(x_true).item()) ** 0.5 / dn) * d
    return x_true + eta * (float(np.linalg.norm(np.asarray(x_true).ravel())) / dn) * draw


def make_dataset(spec, budget=None, device=None):
    """(observed, true_cores) for a spec (synthetic.py:184-197): independent child
    streams for the cores and the noise, the dense tensor reconstructed on the GPU.

    device=None returns the observed tensor as a host array (the reference's
    return type); a CUDA device keeps it resident there (no D2H)."""
    spec.validate()
    check_element_budget([spec.dim] * spec.order, budget)
    core_seed, noise_seed = spawn_seeds(spec.seed, 2)
    cores = _GENERATORS[spec.kind](spec, rng=make_rng(core_seed))
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_11362_b200.make_dataset reconstructs on the GPU (no CPU path)")
    x_true = reconstruct_device(cores, device=device if device is not None else "cuda")
    if device is None:
        x_true = x_true.cpu().numpy()
    return add_noise(x_true, spec.noise, rng=make_rng(noise_seed)), cores


def _stream():
    return int(torch.cuda.current_stream().cuda_stream)


def reconstruct_device(cores, device="cuda") -> torch.Tensor:
    """Dense tensor of a ring (C-order cores) on the device: X[pre][post] = sum HL[pre][a][b] HR[post][b][a]."""
    lib = L.lib()
    cs = [torch.as_tensor(np.asarray(g, dtype=np.float64)).to(device).contiguous() for g in cores]
    N = len(cs)
    if N < 2:
        raise ValueError("reconstruct needs at least two cores")
    dims = [int(g.shape[1]) for g in cs]
    ranks = [int(g.shape[0]) for g in cs]
    h = N // 2
    sp = _stream()

    def chain(lo, hi, transposed):
        blk = list(range(lo, hi + 1))
        bd = [dims[j] for j in blk]
        br = [ranks[j % N] for j in range(lo, hi + 2)]
        first = torch.empty((bd[0], br[0], br[1]), dtype=torch.float64, device=device)
        L.check(lib.trals_core_relayout_f64(cs[lo].data_ptr(), L.LAYOUT_C, br[0], bd[0], br[1], first.data_ptr(),
                                            L.LAYOUT_SLICE, sp), "relayout")
        n = int(np.prod(bd)) * br[0] * br[-1]
        out = torch.empty(n, dtype=torch.float64, device=device)
        tmp = torch.empty(max(1, lib.trals_half_chain_tmp_elems(len(blk), L.i64_array(bd), L.i32_array(br))),
                          dtype=torch.float64, device=device)
        need = 1
        pre = bd[0]
        for j in range(1, len(blk)):
            need = max(need, lib.trals_gemm_ws_elems(1, pre * br[0], br[j], bd[j] * br[j + 1]))
            pre *= bd[j]
        ws = torch.empty(need, dtype=torch.float64, device=device)
        L.check(lib.trals_half_chain_f64(len(blk), L.i64_array(bd), L.i32_array(br), first.data_ptr(),
                                         L.ptr_array([cs[j].data_ptr() for j in blk]), out.data_ptr(),
                                         tmp.data_ptr(), ws.data_ptr(), ws.numel(), transposed, sp), "half_chain")
        return out, int(np.prod(bd))

    HL, pre = chain(0, h - 1, 0)   # [pre][r_0][r_h]
    B, post = chain(h, N - 1, 1)   # [r_0][r_h][post]
    R0, Rh = ranks[0], ranks[h]
    X = torch.empty(dims, dtype=torch.float64, device=device)
    K = R0 * Rh
    need = lib.trals_gemm_ws_elems(1, pre, K, post)
    ws = torch.empty(max(need, 1), dtype=torch.float64, device=device)
    L.check(lib.trals_gemm_f64(HL.data_ptr(), 0, K, 1, 1, pre, K, post, B.data_ptr(), post, X.data_ptr(),
                               L.i64_array([0, 1 << 40, 0, post, 1 << 40, 0, 1]), 0, ws.data_ptr(), ws.numel(), sp),
            "reconstruct gemm")
    return X


def _sumsq(x):
    lib = L.lib()
    out = torch.empty(2, dtype=torch.float64, device=x.device)
    ws = torch.empty(lib.trals_sumsq_ws_elems(), dtype=torch.float64, device=x.device)
    L.check(lib.trals_sumsq_f64(x.data_ptr(), x.numel(), out.data_ptr(), ws.data_ptr(), _stream()), "sumsq")
    return out[:1]


def make_dataset_device(order, dim, rank, noise, seed, device="cuda", noise_source="device"):
    """(x on the device, true cores on the host) for a cubic gaussian recipe."""
    core_seed, noise_seed = spawn_seeds(seed, 2)
    rng = make_rng(core_seed)
    cores = [rng.standard_normal((rank, dim, rank)) for _ in range(order)]
    x = reconstruct_device(cores, device=device)
    if noise > 0:
        if noise_source == "host":
            draw = torch.from_numpy(make_rng(noise_seed).standard_normal(x.shape)).to(device)
        else:
            g = torch.Generator(device=device)
            g.manual_seed(int(noise_seed.generate_state(1, np.uint64)[0] & ((1 << 63) - 1)))
            draw = torch.randn(x.shape, dtype=torch.float64, device=device, generator=g)
        scale = noise * float(_sumsq(x).item()) ** 0.5 / float(_sumsq(draw).item()) ** 0.5
        x.add_(draw, alpha=scale)
        del draw
    return x, cores
