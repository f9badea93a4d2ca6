"""Numpy model of the libtrals C-ABI -- TEST INFRASTRUCTURE ONLY.

Implements every entry point of include/trals.h from its documented
semantics (independently of the CUDA code), operating on raw host pointers
(CPU torch tensors).  Injected into `SweepEngine(_test_lib=FakeTrals())`, it
lets the CPU test suite execute the engine's exact step list -- the
environment-tree schedule, the index conventions, the shard/all-reduce logic
-- and compare the sweep with the oracle without a GPU.  It is never used by
the product path.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.linalg as sla


def _arr(ptr, n):
    ptr = int(ptr.value if isinstance(ptr, ctypes.c_void_p) else ptr)
    return np.ctypeslib.as_array((ctypes.c_double * int(n)).from_address(ptr))


def _farr(ptr, n):
    ptr = int(ptr.value if isinstance(ptr, ctypes.c_void_p) else ptr)
    return np.ctypeslib.as_array((ctypes.c_float * int(n)).from_address(ptr))


def _i8arr(ptr, n):
    ptr = int(ptr.value if isinstance(ptr, ctypes.c_void_p) else ptr)
    return np.ctypeslib.as_array((ctypes.c_int8 * int(n)).from_address(ptr))


def _i32arr(ptr, n):
    ptr = int(ptr.value if isinstance(ptr, ctypes.c_void_p) else ptr)
    return np.ctypeslib.as_array((ctypes.c_int32 * int(n)).from_address(ptr))


def oz_digits_bytes(rows, k, rows_per_tile=128):
    """Bytes of the tiled int8 digit layout (include/trals.h, trals_oz_digits_bytes)."""
    return 4 * (-(-rows // rows_per_tile) * rows_per_tile) * (-(-k // 64) * 64)


def oz_offsets(rows, k, plane, rows_per_tile=128, digits=4, bk=64):
    """Byte offsets [rows, k] of one digit plane in the tiled layout
    [row tile][bk-k block][plane][rows_per_tile x bk B]: SWIZZLE_64B rows (bk 64, chunk c of
    row r at c ^ ((r >> 1) & 3)) or SWIZZLE_32B rows (bk 32, chunk c at c ^ ((r >> 2) & 1))."""
    r = np.arange(rows, dtype=np.int64)[:, None]
    kk = np.arange(k, dtype=np.int64)[None, :]
    kblocks = -(-k // bk)
    t, rr, kb, c = r // rows_per_tile, r % rows_per_tile, kk // bk, kk % bk
    block = (t * kblocks + kb) * digits + plane
    sw = ((c >> 4) ^ ((rr >> 1) & 3)) if bk == 64 else ((c >> 4) ^ ((rr >> 2) & 1))
    return block * rows_per_tile * bk + rr * bk + (sw << 4) + (c & 15)


def oz_slice(v):
    """Row exponents (|x| < 2^e) and four truncated base-128 digit planes of v [rows, k]."""
    mx = np.max(np.abs(v), axis=1)
    e = np.where(mx > 0, np.frexp(mx)[1], 0).astype(np.int32)
    w = np.ldexp(v, -e[:, None].astype(np.int64))
    planes = []
    for _ in range(4):
        t = w * 128.0
        q = np.trunc(t)
        planes.append(q.astype(np.int8))
        w = t - q
    return planes, e


def _iarr(ptr, n):
    ptr = int(ptr.value if isinstance(ptr, ctypes.c_void_p) else ptr)
    return np.ctypeslib.as_array((ctypes.c_int32 * int(n)).from_address(ptr))


def _vals(a, n):
    return [int(a[i]) for i in range(n)]


def _ptrs(a, n):
    return [int(a[i]) for i in range(n)]


class FakeTrals:
    def __init__(self):
        self.calls = {}

    def _count(self, name):
        self.calls[name] = self.calls.get(name, 0) + 1

    # --- helpers ---------------------------------------------------------
    def trals_strerror(self, code):
        return b"fake"

    def trals_version(self):
        return 1

    def trals_gemm_ws_elems(self, P, M, K, N):
        return 0

    def trals_sumsq_ws_elems(self):
        return 4

    def trals_error_ws_elems(self, rows, m):
        return 1

    def trals_half_chain_tmp_elems(self, nblk, dims, ranks):
        return 1

    # --- generic GEMM ----------------------------------------------------
    def trals_gemm_f64(self, A, sAp, sAm, sAk, P, M, K, N, B, ldb, C, cmap, beta, ws, ws_elems, stream):
        self._count("gemm")
        cm = [int(cmap[i]) for i in range(7)]
        amax = (P - 1) * sAp + (M - 1) * sAm + (K - 1) * sAk + 1
        a = _arr(A, amax)
        av = np.lib.stride_tricks.as_strided(a, shape=(P, M, K), strides=(sAp * 8, sAm * 8, sAk * 8))
        b = _arr(B, (K - 1) * ldb + N)
        bv = np.lib.stride_tricks.as_strided(b, shape=(K, N), strides=(ldb * 8, 8))
        res = np.einsum("pmk,kn->pmn", av, bv)
        p = np.arange(P)[:, None, None]
        m = np.arange(M)[None, :, None]
        n = np.arange(N)[None, None, :]
        addr = p * cm[0] + (m // cm[1]) * cm[2] + (m % cm[1]) * cm[3] + (n // cm[4]) * cm[5] + (n % cm[4]) * cm[6]
        c = _arr(C, int(addr.max()) + 1)
        if beta:
            c[addr] += res
        else:
            c[addr] = res
        return 0

    # --- layouts ---------------------------------------------------------
    @staticmethod
    def _to_canon(buf, layout, Ra, I, Rb):
        if layout == 0:
            return buf.reshape(Ra, I, Rb)
        if layout == 1:
            return buf.reshape(I, Ra, Rb).transpose(1, 0, 2)
        return buf.reshape(I, Rb, Ra).transpose(2, 0, 1)

    @staticmethod
    def _from_canon(g, layout):
        if layout == 0:
            return g
        if layout == 1:
            return g.transpose(1, 0, 2)
        return g.transpose(1, 2, 0)

    def trals_core_relayout_f64(self, src, sl, Ra, I, Rb, dst, dl, stream):
        self._count("relayout")
        n = Ra * I * Rb
        g = self._to_canon(_arr(src, n).copy(), sl, Ra, I, Rb)
        _arr(dst, n)[:] = np.ascontiguousarray(self._from_canon(g, dl)).ravel()
        return 0

    # --- ring pieces -----------------------------------------------------
    def trals_half_chain_f64(self, nblk, dims, ranks, first_slice, cores_c, out, tmp, ws, ws_elems, transposed,
                             stream):
        self._count("half_chain")
        d = _vals(dims, nblk)
        r = _vals(ranks, nblk + 1)
        cc = _ptrs(cores_c, nblk) if nblk > 1 else []
        h = _arr(first_slice, d[0] * r[0] * r[1]).reshape(d[0], r[0], r[1]).copy()
        for j in range(1, nblk):
            g = _arr(cc[j], r[j] * d[j] * r[j + 1]).reshape(r[j], d[j], r[j + 1])
            h = np.einsum("pat,tic->piac", h, g).reshape(-1, r[0], r[j + 1])
        if transposed:
            h = np.ascontiguousarray(h.transpose(2, 1, 0))
        _arr(out, h.size)[:] = h.ravel()
        return 0

    def trals_residual_ws_elems(self, pre, post):
        return 1

    def trals_residual_oz64_ws_elems(self, pre, post, K):
        return 1

    def trals_residual_oz64(self, X, pre, post, HL, HRt, K, xnorm2, out, ws, ws_elems, stream):
        # same quantity as trals_residual_f64 (the int8 product is fp64-accurate)
        return self.trals_residual_f64(X, pre, post, HL, HRt, K, xnorm2, out, ws, ws_elems, stream)

    def trals_residual_f64(self, X, pre, post, HL, HRt, K, xnorm2, out, ws, ws_elems, stream):
        self._count("residual")
        x = _arr(X, pre * post).reshape(pre, post)
        hl = _arr(HL, pre * K).reshape(pre, K)
        hr = _arr(HRt, K * post).reshape(K, post)
        ssr = float(np.sum((x - hl @ hr) ** 2))
        x2 = float(_arr(xnorm2, 1)[0])
        o = _arr(out, 3)
        o[1] = ssr
        o[0] = 0.0 if x2 == 0 else np.sqrt(ssr / x2)
        return 0

    # --- fp32 variant: the 3xTF32 split and the K-major environment product ---
    def trals_oz_digits_bytes(self, rows, k):
        return oz_digits_bytes(rows, k)

    def trals_oz_split_ws_elems(self, rows, cols, transpose):
        return cols if transpose else rows

    def trals_oz_split_f32(self, x, rows, cols, transpose, digits, exps, ws, ws_elems, stream):
        self._count("oz_split")
        v = _farr(x, rows * cols).reshape(rows, cols).astype(np.float64)
        if transpose:
            v = v.T
        r, k = v.shape
        planes, e = oz_slice(v)
        buf = _i8arr(digits, oz_digits_bytes(r, k))
        buf[:] = 0
        for s in range(4):
            buf[oz_offsets(r, k, s)] = planes[s]
        _i32arr(exps, r)[:] = e
        return 0

    def trals_env_oz_ws_elems(self, pre, post, side, r_lo, r_hi):
        return 1

    def trals_env_oz(self, xd, xe, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems, stream):
        rows, k = (pre, post) if side == 0 else (post, pre)
        buf = _i8arr(xd, oz_digits_bytes(rows, k))
        e = _i32arr(xe, rows).astype(np.int64)
        a = sum(buf[oz_offsets(rows, k, s)].astype(np.float64) * 2.0 ** (-7 * (s + 1)) for s in range(4))
        a = np.ldexp(a, e[:, None])
        x = np.ascontiguousarray(a if side == 0 else a.T)
        return self.trals_env_f64(x.ctypes.data, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems, stream)

    def trals_sumsq_f32(self, x, n, out, ws, stream):
        self._count("sumsq")
        v = _farr(x, n).astype(np.float64)
        o = _arr(out, 2)
        o[0] = float(np.dot(v, v))
        o[1] = float(np.count_nonzero(~np.isfinite(v)))
        return 0

    def trals_env_f64(self, X, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems, stream):
        self._count("env")
        x = _arr(X, pre * post).reshape(pre, post)
        if side == 0:
            h = _arr(H, post * r_lo * r_hi).reshape(post, r_lo, r_hi)   # [k][r_y][r_0]
            env = np.einsum("mk,kyz->zmy", x, h)                         # [r_0][m][r_y]
            if leaf:  # M_0[i][r_0 + R_0 r_1]
                out = env.transpose(1, 2, 0).reshape(pre, -1)          # [m][r_y][r_0]
            else:
                out = env
        else:
            h = _arr(H, pre * r_lo * r_hi).reshape(pre, r_lo, r_hi)    # [k][r_0][r_x1]
            env = np.einsum("km,kzx->xmz", x, h)                         # [r_x1][m][r_0]
            if leaf:  # M_{N-1}[i][r_{N-1} + R_{N-1} r_0]
                out = env.transpose(1, 2, 0).reshape(post, -1)
            else:
                out = env
        _arr(E, out.size)[:] = np.ascontiguousarray(out).ravel()
        return 0

    def trals_absorb_right_f64(self, E, Ra, pre, Ib, Rb, Rb1, core_zt, out, leaf, ws, ws_elems, stream):
        self._count("absorb_right")
        e = _arr(E, Ra * pre * Ib * Rb1).reshape(Ra, pre, Ib, Rb1)
        gt = _arr(core_zt, Ib * Rb1 * Rb).reshape(Ib, Rb1, Rb)
        o = np.einsum("apir,irb->apb", e, gt)                           # [r_a][pre][r_b]
        if leaf:
            o = o.transpose(1, 2, 0).reshape(pre, Rb * Ra)              # [i_a][r_b][r_a]
        _arr(out, o.size)[:] = np.ascontiguousarray(o).ravel()
        return 0

    def trals_absorb_left_f64(self, E, Ra, Ia, rest, Ra1, Rb1, core_c, out, leaf, ws, ws_elems, stream):
        self._count("absorb_left")
        e = _arr(E, Ra * Ia * rest * Rb1).reshape(Ra, Ia, rest, Rb1)
        g = _arr(core_c, Ra * Ia * Ra1).reshape(Ra, Ia, Ra1)
        o = np.einsum("airz,aic->crz", e, g)                            # [r_a1][rest][r_b1]
        if leaf:
            o = o.transpose(1, 2, 0).reshape(rest, Rb1 * Ra1)           # [i_b][r_b1][r_b]
        _arr(out, o.size)[:] = np.ascontiguousarray(o).ravel()
        return 0

    def trals_core_gram_f64(self, Gs, Ra, I, Rb, E, ws, ws_elems, stream):
        self._count("core_gram")
        g = _arr(Gs, I * Ra * Rb).reshape(I, Ra, Rb)
        e = np.einsum("iab,icd->acbd", g, g).reshape(Ra * Ra, Rb * Rb)
        _arr(E, e.size)[:] = e.ravel()
        return 0

    def trals_core_qr_ws_elems(self, I, RR):
        return 1

    def trals_core_qr_f64(self, Gzt, I, RR, R, ws, ws_elems, stream):
        self._count("core_qr")
        g = _arr(Gzt, I * RR).reshape(I, RR)
        r = np.linalg.qr(g, mode="r")
        sg = np.sign(np.diagonal(r)).copy()
        sg[sg == 0] = 1.0
        r = r * sg[:, None]
        _arr(R, r.size)[:] = r.ravel()
        return 0

    def trals_gram_chain_part_f64(self, N, n, ranks, E, S, tmp, ws, ws_elems, part, stream):
        """part 1 (prefix) is a no-op in this model; part 2 / 0 form the whole chain."""
        if part == 1:
            self._count("gram_chain_prefix")
            return 0
        return self.trals_gram_chain_f64(N, n, ranks, E, S, tmp, ws, ws_elems, stream)

    def trals_gram_chain_f64(self, N, n, ranks, E, S, tmp, ws, ws_elems, stream):
        self._count("gram_chain")
        r = _vals(ranks, N)
        es = _ptrs(E, N)
        order = list(range(n + 1, N)) + list(range(n))
        F = None
        for j in order:
            Rj, Rj1 = r[j], r[(j + 1) % N]
            e = _arr(es[j], Rj * Rj * Rj1 * Rj1).reshape(Rj * Rj, Rj1 * Rj1)
            F = e.copy() if F is None else F @ e
        Rn, Rn1 = r[n], r[(n + 1) % N]
        f = F.reshape(Rn1, Rn1, Rn, Rn)                                  # [x][y][b][d]
        s = f.transpose(0, 2, 1, 3)  # [x][b][y][d]: row (x, b) = b + Rn*x, col (y, d) = d + Rn*y
        s = s.reshape(Rn1 * Rn, Rn1 * Rn)
        _arr(S, s.size)[:] = s.ravel()
        return 0

    def trals_cholesky_aux_elems(self, m):
        return 1

    def trals_chol_solve_ws_elems(self, rows, m):
        return 1

    def trals_cholesky_f64(self, S, m, U, Lo, aux, check_degen, info, stream):
        self._count("cholesky")
        s = _arr(S, m * m).reshape(m, m)
        inf = _iarr(info, 6)
        scale = np.max(np.abs(s))
        if scale > 0 and np.max(np.abs(s - s.T)) > 1e-8 * scale:
            inf[1] = 1
        sym = 0.5 * (s + s.T)
        try:
            u = sla.cholesky(sym, lower=False)
        except np.linalg.LinAlgError:
            inf[0] = 1
            return 0
        _arr(U, m * m)[:] = u.ravel()
        _arr(Lo, m * m)[:] = u.T.ravel()
        if check_degen:
            d = np.abs(np.diagonal(u))
            if d.min() <= 1e-13 * np.max(np.abs(u)):
                inf[2] = int(np.argmin(d)) + 1
        return 0

    def trals_chol_solve_f64(self, U, Lo, aux, m, M, rows, Z, ws, ws_elems, stream):
        self._count("chol_solve")
        u = _arr(U, m * m).reshape(m, m)
        rhs = _arr(M, rows * m).reshape(rows, m)
        try:
            y = sla.solve_triangular(u, rhs.T, trans="T", lower=False)
            z = sla.solve_triangular(u, y, lower=False).T
        except np.linalg.LinAlgError:  # singular R0: the device solve writes non-finite values here,
            z = np.full((rows, m), np.nan)  # which the fallback step that follows overwrites
        _arr(Z, rows * m)[:] = z.ravel()
        return 0

    def trals_solve_refine_f64(self, F, aux, S, m, M, rows, Z, info, stream):
        self._count("refine")  # the numpy model's solve is already a backward-stable triangular solve
        return 0

    def trals_spd_fallback_ws_elems(self, rows, m):
        return 1

    def trals_spd_fallback_f64(self, S, m, M, rows, Z, info, mode, rcond, ws, ws_elems, stream):
        self._count("fallback")
        inf = _iarr(info, 6)
        fire = inf[0] != 0 if mode == 0 else (inf[0] != 0 or inf[2] != 0 if mode == 1 else True)
        if not fire:
            return 0
        s = _arr(S, m * m).reshape(m, m)
        sym = 0.5 * (s + s.T)
        rhs = _arr(M, rows * m).reshape(rows, m)
        nf = m * 2.220446049250313e-16
        cut = max(rcond, nf) if mode == 0 else max(rcond * rcond, nf)
        u, sig, vt = np.linalg.svd(sym)
        keep = sig > cut * sig[0]
        pinv = (vt[keep].T / sig[keep]) @ u[:, keep].T
        _arr(Z, rows * m)[:] = (rhs @ pinv).ravel()
        if mode != 2:
            inf[0] = 0
            if mode == 1:
                inf[2] = 0
            inf[3] += 1
        return 0

    def trals_dd_transfer_f64(self, Rc, Ra, k, Rb, Ehi, Elo, stream):
        """Transfer matrix of one tensor in extended precision (the dd planes' semantics)."""
        self._count("dd_transfer")
        r = _arr(Rc, Ra * k * Rb).reshape(Ra, k, Rb).astype(np.longdouble)
        e = np.einsum("aib,cid->acbd", r, r).reshape(Ra * Ra, Rb * Rb)
        hi = e.astype(np.float64)
        _arr(Ehi, e.size)[:] = hi.ravel()
        _arr(Elo, e.size)[:] = (e - hi).astype(np.float64).ravel()
        return 0

    def trals_dd_r0_ws_elems(self, N, ranks):
        return 1

    def trals_dd_r0_f64(self, N, n, ranks, Ehi, Elo, S, R0, ws, ws_elems, stream):
        """S_n from the transfer matrices and its semidefinite Cholesky factor, in extended precision."""
        self._count("dd_r0")
        r = _vals(ranks, N)
        hs, ls = _ptrs(Ehi, N), _ptrs(Elo, N)
        order = list(range(n + 1, N)) + list(range(n))
        F = None
        for j in order:
            Rj, Rj1 = r[j], r[(j + 1) % N]
            sz = Rj * Rj * Rj1 * Rj1
            e = (_arr(hs[j], sz).astype(np.longdouble) + _arr(ls[j], sz).astype(np.longdouble)).reshape(
                Rj * Rj, Rj1 * Rj1)
            F = e.copy() if F is None else F @ e
        Rn, Rn1 = r[n], r[(n + 1) % N]
        s = F.reshape(Rn1, Rn1, Rn, Rn).transpose(0, 2, 1, 3).reshape(Rn1 * Rn, Rn1 * Rn)
        m = s.shape[0]
        if S:
            _arr(S, m * m)[:] = s.astype(np.float64).ravel()
        w = s.copy()
        u = np.zeros((m, m), dtype=np.longdouble)
        for j in range(m):
            d = w[j, j]
            if d > 0:
                u[j, j:] = w[j, j:] / np.sqrt(d)
                w[j + 1:, j + 1:] -= np.outer(u[j, j + 1:], u[j, j + 1:])
        _arr(R0, m * m)[:] = u.astype(np.float64).ravel()
        return 0

    def trals_tri_prepare_f64(self, U, m, F, aux, check_degen, info, stream):
        self._count("tri_prepare")
        u = np.triu(_arr(U, m * m).reshape(m, m))
        _arr(U, m * m)[:] = u.ravel()
        _arr(F, m * m)[:] = u.T.ravel()
        if check_degen:
            d = np.abs(np.diagonal(u))
            if d.min() <= 1e-13 * np.max(np.abs(u)):
                _iarr(info, 6)[2] = int(np.argmin(d)) + 1
            if d.min() <= np.sqrt(m * 2.220446049250313e-16) * np.max(np.abs(u)):
                _iarr(info, 6)[4] = 1
        return 0

    def trals_tri_fallback_f64(self, R0, Lr, m, M, rows, Z, info, mode, rcond, ws, ws_elems, stream):
        self._count("fallback")
        inf = _iarr(info, 6)
        fire = {1: inf[2] != 0 or inf[4] != 0, 2: True, 3: inf[4] != 0}[mode]
        if not fire:
            return 0
        counted = mode == 1 and inf[2] != 0
        r0 = _arr(R0, Lr * m).reshape(Lr, m)
        rhs = _arr(M, rows * m).reshape(rows, m)
        _, sig, vt = np.linalg.svd(r0, full_matrices=False)
        keep = sig > max(rcond, np.sqrt(m * 2.220446049250313e-16)) * sig[0]
        v = vt[keep].T
        _arr(Z, rows * m)[:] = (((rhs @ v) / sig[keep] ** 2) @ v.T).ravel()
        if mode == 1:
            inf[2] = 0
        inf[4] = 0
        if counted:
            inf[3] += 1
        return 0

    def trals_sumsq_f64(self, x, n, out, ws, stream):
        self._count("sumsq")
        v = _arr(x, n)
        o = _arr(out, 2)
        o[0] = float(np.dot(v, v))
        o[1] = float(np.count_nonzero(~np.isfinite(v)))
        return 0

    def trals_error_terms_f64(self, M, Z, S, rows, m, xnorm2, out, ws, ws_elems, stream):
        self._count("error_terms")
        mm = _arr(M, rows * m).reshape(rows, m)
        z = _arr(Z, rows * m).reshape(rows, m)
        s = _arr(S, m * m).reshape(m, m)
        cross = float(np.vdot(mm, z))
        model = float(np.vdot(s, z.T @ z))
        x2 = float(_arr(xnorm2, 1)[0])
        xn = np.sqrt(x2)
        e = 0.0 if xn == 0 else np.sqrt(max(0.0, xn * xn - 2 * cross + model)) / xn
        o = _arr(out, 3)
        o[0], o[1], o[2] = e, cross, model
        return 0
