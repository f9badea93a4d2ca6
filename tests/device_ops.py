"""TEST SUPPORT: tensor-level wrappers over the C-ABI (torch tensors in, torch tensors out).

The device operators the sweep engine is built from, exposed one by one so
the operator-level parity tests (tests/test_gpu_ops.py) can check each
against the oracle.  All inputs must be CUDA float64 tensors; nothing here
falls back to the CPU.  Not part of the product package.
"""

from __future__ import annotations

import torch

from paper_2210_11362_b200 import _lib as L


def _stream():
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(stream):
    return int(stream.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
            raise TypeError("libtrals operators take CUDA float64 tensors")
        if not t.is_contiguous():
            raise ValueError("libtrals operators take contiguous tensors")


def ws(elems: int, device) -> torch.Tensor:
    return torch.empty(max(int(elems), 1), dtype=torch.float64, device=device)


def relayout(core: torch.Tensor, src: int, dst: int, shape) -> torch.Tensor:
    """Move a core between the C / SLICE / ZT layouts (see include/trals.h)."""
    _require_cuda(core)
    ra, i, rb = (int(v) for v in shape)
    out_shape = {L.LAYOUT_C: (ra, i, rb), L.LAYOUT_SLICE: (i, ra, rb), L.LAYOUT_ZT: (i, rb, ra)}[dst]
    out = torch.empty(out_shape, dtype=torch.float64, device=core.device)
    L.check(L.lib().trals_core_relayout_f64(core.data_ptr(), src, ra, i, rb, out.data_ptr(), dst, _stream()),
            "trals_core_relayout_f64")
    return out


def core_layouts(core_c: torch.Tensor):
    """(C, SLICE, ZT) device copies of a C-order core."""
    shape = core_c.shape
    return core_c, relayout(core_c, L.LAYOUT_C, L.LAYOUT_SLICE, shape), relayout(core_c, L.LAYOUT_C, L.LAYOUT_ZT, shape)


def gemm(A, sAp, sAm, sAk, P, M, K, N, B, ldb, C, cmap, beta=0):
    need = L.lib().trals_gemm_ws_elems(P, M, K, N)
    w = ws(need, A.device)
    L.check(L.lib().trals_gemm_f64(A.data_ptr(), sAp, sAm, sAk, P, M, K, N, B.data_ptr(), ldb, C.data_ptr(),
                                   L.i64_array(cmap), beta, w.data_ptr(), w.numel(), _stream()),
            "trals_gemm_f64")
    return C


def mttsp(x: torch.Tensor, cores_c, n: int) -> torch.Tensor:
    """M_n = X_[n] G^{!=n}_[2] (reference solvers.py:375,379) for one mode."""
    _require_cuda(x, *cores_c)
    N = x.dim()
    dims = list(x.shape)
    ranks = [int(g.shape[0]) for g in cores_c]
    lay = [core_layouts(g) for g in cores_c]
    dims_a, ranks_a = L.i64_array(dims), L.i32_array(ranks)
    need = L.lib().trals_mttsp_ws_elems(N, dims_a, ranks_a, n)
    w = ws(need, x.device)
    rr = ranks[n] * ranks[(n + 1) % N]
    out = torch.empty((dims[n], rr), dtype=torch.float64, device=x.device)
    st = L.lib().trals_mttsp_f64(
        x.data_ptr(), N, dims_a, ranks_a, n,
        L.ptr_array([c.data_ptr() for c, _, _ in lay]),
        L.ptr_array([s.data_ptr() for _, s, _ in lay]),
        L.ptr_array([z.data_ptr() for _, _, z in lay]),
        out.data_ptr(), w.data_ptr(), w.numel(), _stream())
    L.check(st, "trals_mttsp_f64")
    return out


def transfer_matrix(core_c: torch.Tensor) -> torch.Tensor:
    """E[(a,c),(b,d)] = sum_i G[a,i,b] G[c,i,d] (the bond Gram of ring.py:173-188)."""
    _require_cuda(core_c)
    ra, i, rb = (int(v) for v in core_c.shape)
    gs = relayout(core_c, L.LAYOUT_C, L.LAYOUT_SLICE, core_c.shape)
    e = torch.empty((ra * ra, rb * rb), dtype=torch.float64, device=core_c.device)
    need = L.lib().trals_gemm_ws_elems(1, ra * rb, i, ra * rb)
    w = ws(need, core_c.device)
    L.check(L.lib().trals_core_gram_f64(gs.data_ptr(), ra, i, rb, e.data_ptr(), w.data_ptr(), w.numel(), _stream()),
            "trals_core_gram_f64")
    return e


def coefficient_gram(cores_c, n: int) -> torch.Tensor:
    """S_n via the transfer-matrix chain (ring.py:191-214, Prop. 3)."""
    N = len(cores_c)
    ranks = [int(g.shape[0]) for g in cores_c]
    es = [transfer_matrix(g) for g in cores_c]
    rr = ranks[n] * ranks[(n + 1) % N]
    rmax = max(ranks)
    S = torch.empty((rr, rr), dtype=torch.float64, device=cores_c[0].device)
    tmp = ws(2 * rmax ** 4, S.device)
    need = max(L.lib().trals_gemm_ws_elems(1, rmax * rmax, rmax * rmax, rmax * rmax), 1)
    w = ws(need, S.device)
    L.check(L.lib().trals_gram_chain_f64(N, n, L.i32_array(ranks), L.ptr_array([e.data_ptr() for e in es]),
                                         S.data_ptr(), tmp.data_ptr(), w.data_ptr(), w.numel(), _stream()),
            "trals_gram_chain_f64")
    return S


class CholFactor:
    """Device Cholesky factor: U (upper), companion F (U^{-1} for m <= 112, else U^T), aux, info flags."""

    def __init__(self, U, Lo, aux, info):
        self.U, self.L, self.aux, self.info = U, Lo, aux, info

    def __iter__(self):  # (U, L, info) unpacking
        return iter((self.U, self.L, self.info))


def cholesky(S: torch.Tensor, check_degen: bool = False) -> CholFactor:
    """Upper Cholesky S = U^T U with the reference's checks (linalg.py:55-81)."""
    _require_cuda(S)
    m = int(S.shape[0])
    U = torch.empty_like(S)
    Lo = torch.empty_like(S)
    aux = ws(L.lib().trals_cholesky_aux_elems(m), S.device)
    info = torch.zeros(L.INFO_SLOTS, dtype=torch.int32, device=S.device)
    L.check(L.lib().trals_cholesky_f64(S.data_ptr(), m, U.data_ptr(), Lo.data_ptr(), aux.data_ptr(),
                                       int(check_degen), info.data_ptr(), _stream()), "trals_cholesky_f64")
    return CholFactor(U, Lo, aux, info)


def chol_solve(f: CholFactor, M: torch.Tensor) -> torch.Tensor:
    """Z with Z (U^T U) = M (cho_solve, linalg.py:76)."""
    _require_cuda(f.U, f.L, M)
    m = int(f.U.shape[0])
    rows = int(M.shape[0])
    Z = torch.empty_like(M)
    w = ws(L.lib().trals_chol_solve_ws_elems(rows, m), M.device)
    L.check(L.lib().trals_chol_solve_f64(f.U.data_ptr(), f.L.data_ptr(), f.aux.data_ptr(), m, M.data_ptr(), rows,
                                         Z.data_ptr(), w.data_ptr(), w.numel(), _stream()), "trals_chol_solve_f64")
    return Z


def sumsq(x: torch.Tensor) -> torch.Tensor:
    _require_cuda(x)
    out = torch.empty(2, dtype=torch.float64, device=x.device)
    w = ws(L.lib().trals_sumsq_ws_elems(), x.device)
    L.check(L.lib().trals_sumsq_f64(x.data_ptr(), x.numel(), out.data_ptr(), w.data_ptr(), _stream()),
            "trals_sumsq_f64")
    return out


def error_terms(M, Z, S, xnorm2) -> torch.Tensor:
    """[e, <M,Z>, <S,Z^T Z>] (solvers.py:177-212, NE form)."""
    _require_cuda(M, Z, S, xnorm2)
    rows, m = (int(v) for v in M.shape)
    out = torch.empty(3, dtype=torch.float64, device=M.device)
    w = ws(L.lib().trals_error_ws_elems(rows, m), M.device)
    L.check(L.lib().trals_error_terms_f64(M.data_ptr(), Z.data_ptr(), S.data_ptr(), rows, m, xnorm2.data_ptr(),
                                          out.data_ptr(), w.data_ptr(), w.numel(), _stream()),
            "trals_error_terms_f64")
    return out
