"""Tensor-ring algebra helpers of the reference's public surface (pkg/src/tenring/ring.py), on the GPU.

These sit beside the hot path (the sweep never calls them: it keeps its cores,
transfer matrices and half chains on the device in its own layouts); they exist
so a caller importing them from the reference package finds them here with the
same names, arguments, shapes, index conventions and errors.  Arithmetic runs
on the CUDA device in fp64 (torch tensors; cuBLAS / cuSOLVER behind
torch.einsum, matmul and linalg.qr) -- there is no CPU path -- and results come
back as numpy arrays like the reference's.  Index conventions:

* cores (R_n, I_n, R_{n+1}), lateral slices G(i) = G[:, i, :] (ring.py:1-24);
* merged lateral index j1 + J1 j2, first factor fastest (ring.py:110-131);
* bond Gram P[a, b, c, d] = sum_i g[b, i, a] z[d, i, c] (ring.py:173-188);
* Gram chains contracted with contract_24_13 and split-unfolded, left bond
  fastest (ring.py:191-214, tensor_ops.py:84-97, 206-225).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .host import check_element_budget, random_cores, validate_cores  # noqa: F401  (re-exported)

__all__ = ["Mode2Qr", "gram_chain", "gram_chain_order", "lateral_gram", "mode2_qr", "random_cores", "reconstruct",
           "subchain_merge", "subchain_skip", "tr_inner", "tr_norm", "validate_cores"]


def _dev():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_11362_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _t(a):
    import torch
    if isinstance(a, torch.Tensor):
        return a.detach().to(device=_dev(), dtype=torch.float64)
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=_dev())


def _np(t):
    return t.detach().cpu().numpy()


def _merge(a, b):
    """(I, J1, K) x (K, J2, L) -> (I, J1 J2, L), slice j1 + J1 j2 = a(j1) @ b(j2), on the device."""
    ia, ja, _ = a.shape
    _, jb, ib = b.shape
    prod = (a.reshape(ia * ja, -1) @ b.reshape(b.shape[0], jb * ib)).reshape(ia, ja, jb, ib)
    return prod.permute(0, 2, 1, 3).contiguous().reshape(ia, jb * ja, ib)


def subchain_merge(a, b):
    """Slice-wise merge of two bond-compatible third-order tensors (ring.py:110-131)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim != 3 or b.ndim != 3:
        raise ValueError("subchain_merge expects two third-order tensors")
    if a.shape[2] != b.shape[0]:
        raise ValueError(f"bond mismatch: left tensor ends in {a.shape[2]}, right starts with {b.shape[0]}")
    return _np(_merge(_t(a), _t(b)))


def _order(skip, n_modes):
    return list(range(skip + 1, n_modes)) + list(range(skip))


def _skip_dev(cores_t, skip):
    order = _order(skip, len(cores_t))
    out = cores_t[order[0]]
    for j in order[1:]:
        out = _merge(out, cores_t[j])
    return out


def subchain_skip(cores, skip):
    """All cores except `skip`, merged in ring order skip+1, ..., N-1, 0, ..., skip-1 (ring.py:138-152)."""
    if len(cores) < 2:
        raise ValueError("subchain_skip needs at least two cores")
    return _np(_skip_dev([_t(c) for c in cores], skip))


def reconstruct(cores, budget=None):
    """Dense tensor of a ring (ring.py:155-170), reconstructed on the device by libtrals' half chains
    and one DMMA GEMM (synthetic.reconstruct_device); refuses tensors over the element budget."""
    from .synthetic import reconstruct_device
    cores = validate_cores(cores)
    if len(cores) < 2:
        raise ValueError("reconstruct needs at least two cores")
    dims = tuple(g.shape[1] for g in cores)
    check_element_budget(dims, budget)
    return _np(reconstruct_device(cores, device=_dev()))


def _gram_dev(g, z):
    import torch
    return torch.einsum("bia,dic->abcd", g, z)


def lateral_gram(g, z=None):
    """P[a, b, c, d] = sum_i g[b, i, a] z[d, i, c]  (ring.py:173-188); z=None: the self-Gram."""
    g = np.asarray(g)
    z = g if z is None else np.asarray(z)
    if g.ndim != 3 or z.ndim != 3:
        raise ValueError("lateral_gram expects third-order tensors")
    if g.shape[1] != z.shape[1]:
        raise ValueError(f"lateral size mismatch: {g.shape[1]} vs {z.shape[1]}")
    tg = _t(g)
    return _np(_gram_dev(tg, tg if z is g else _t(z)))


def gram_chain_order(skip, n_modes):
    """n-1, ..., 0, N-1, ..., n+1: the Gram order matching subchain_skip (ring.py:191-198)."""
    return list(range(skip - 1, -1, -1)) + list(range(n_modes - 1, skip, -1))


def _contract_24_13(a, b):
    import torch
    return torch.einsum("imrk,mjks->ijrs", a, b)


def _split_unfold2(t):
    """split_unfold(t, 2) (tensor_ops.py:84-97): first two axes -> rows, first index fastest."""
    s = t.shape
    return t.permute(3, 2, 1, 0).reshape(s[3] * s[2], s[1] * s[0]).T


def gram_chain(grams):
    """Bond Grams composed with contract_24_13 and split-unfolded (ring.py:201-214)."""
    grams = list(grams)
    if not grams:
        raise ValueError("gram_chain needs at least one Gram tensor")
    out = _t(grams[0])
    for p in grams[1:]:
        out = _contract_24_13(out, _t(p))
    return _np(_split_unfold2(out))


@dataclass
class Mode2Qr:
    """Lateral-unfolding QR of a third-order tensor (ring.py:217-233): q (I x k) orthonormal columns,
    r_tensor (R, k, R') with an upper-triangular classical 2-unfolding, k = min(I, R R')."""

    r_tensor: np.ndarray
    q: np.ndarray

    @property
    def r_matrix(self):
        """Triangular factor as a (k, R R') matrix, left bond fastest (classical 2-unfolding)."""
        return _classical_unfold1(self.r_tensor)


def _classical_unfold1(t):
    """classical_unfold(t, 1) (tensor_ops.py:52-66): rows = axis 1, columns (axis 0, axis 2), axis 0 fastest."""
    return np.asarray(t).transpose(1, 0, 2).reshape(t.shape[1], -1, order="F")


def mode2_qr(g):
    """QR of a core along its lateral mode (ring.py:236-249; nonnegative diag(R), linalg.py:36-52),
    computed on the device."""
    import torch
    g = np.asarray(g, dtype=np.float64)
    if g.ndim != 3:
        raise ValueError("mode2_qr expects a third-order tensor")
    r0, i, r1 = g.shape
    a = _t(_classical_unfold1(g))
    q, r = torch.linalg.qr(a, mode="reduced")
    sgn = torch.sign(torch.diagonal(r))
    sgn[sgn == 0] = 1.0
    q = q * sgn
    r = r * sgn[:, None]
    k = r.shape[0]
    rn = _np(r)
    r_tensor = rn.reshape(k, r0, r1, order="F").transpose(1, 0, 2).copy()
    return Mode2Qr(r_tensor=r_tensor, q=_np(q))


def tr_inner(a_cores, b_cores):
    """<A, B> of two rings without materialising them (ring.py:252-275): cross Grams composed over
    modes N-1, ..., 0, both bond rings closed."""
    import torch
    a_cores = validate_cores(a_cores)
    b_cores = validate_cores(b_cores)
    if len(a_cores) != len(b_cores):
        raise ValueError("rings have different numbers of modes")
    dims_a = tuple(g.shape[1] for g in a_cores)
    dims_b = tuple(g.shape[1] for g in b_cores)
    if dims_a != dims_b:
        raise ValueError(f"mode size mismatch: {dims_a} vs {dims_b}")
    out = _gram_dev(_t(a_cores[-1]), _t(b_cores[-1]))
    for n in range(len(a_cores) - 2, -1, -1):
        out = _contract_24_13(out, _gram_dev(_t(a_cores[n]), _t(b_cores[n])))
    return float(torch.einsum("aacc->", out).item())


def tr_norm(cores):
    """Frobenius norm of a ring (ring.py:278-284); the self inner product is clamped at 0."""
    return math.sqrt(max(0.0, tr_inner(cores, cores)))
