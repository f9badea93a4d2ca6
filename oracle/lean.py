"""Memory-lean CPU oracle for the BASELINE c5 goldens -- TEST INFRASTRUCTURE ONLY.

The reference's own operation order (oracle/tenring_oracle.py) materialises, per
mode update, the subchain unfolding A_n (c5: 4.1M x 400 = 13.1 GB), N unfolded
copies of X (21 GB) and, for TR-ALS-QR, V_[2] and its Q0 (13 GB each).  That
does not fit the 62 GB build container, so this module restates the SAME
algorithms with the big products blocked over the slowest column index of
the cyclic unfolding (the lateral index of mode n-1):

* MTTSP  `X_[n] @ A_n`  (solvers.py:379)  = sum over i_{n-1} of
  `X_[n][:, block] @ unfold(P * G_{n-1}[:, i_{n-1}, :])`, P the subchain of the
  other N-2 cores (ring.py:110-152 for the merge convention);
* QRNE   `Y_[n] @ V_[2]` (solvers.py:480-484), blocked the same way over k_{n-1};
* QR     `qr(V_[2])` (solvers.py:424, linalg.py:36-52) as a two-level TSQR
  (Householder QR of every block, then of the stacked block R factors, signs
  fixed to a nonnegative diagonal), `W = Y_[n] Q0` (solvers.py:431) accumulated
  block by block from the implicit Q0 = diag(Q_c) Q2;
* exact error `||X - reconstruct(G)|| / ||X||` (solvers.py:164-174,
  ring.py:155-170) and the data recipe `make_dataset` (synthetic.py:184-197)
  reconstructed slab by slab along the last mode.

Everything R^2-sized (Gram chains, solves, per-core QR, error terms) calls the
oracle functions unchanged.  Only summation order differs from the reference
(blocked GEMMs, a TSQR instead of one Householder QR), i.e. results agree to
rounding; `tests/test_oracle_golden.py::test_lean_*` pins this module against the
reference's own goldens on c2 (NE + QR, 20 sweeps) and the small rings.

Who may use it: tests/ (and the golden generator tests/golden/make_c5_golden.py),
bench.py's CPU legs.  Never the product package.
"""

from __future__ import annotations

import math

import numpy as np

from . import tenring_oracle as O


# ---------------------------------------------------------------------------
# blocked building blocks
# ---------------------------------------------------------------------------
def _slow_mode(n, N):
    """The mode whose lateral index is the slowest column index of X_[n] (tensor_ops.py:69-81)."""
    return (n - 1) % N


def _x_block_unfold(x, n, c):
    """X_[n][:, columns with i_{n-1} = c] -- the cyclic unfolding of the slice x[i_{n-1} = c]."""
    N = x.ndim
    m = _slow_mode(n, N)
    idx = [slice(None)] * N
    idx[m] = c
    xc = x[tuple(idx)]  # a view; the unfolding below makes the one copy
    nn = n if m > n else n - 1  # index of mode n inside the slice
    return O.unfold_cyclic(xc, nn)


def _prefix_chain(cores, n):
    """Subchain of every core except n and n-1 (ring.py:138-152 order n+1, ..., n-2)."""
    order = O.ring_order_without(n, len(cores))[:-1]
    acc = cores[order[0]]
    for j in order[1:]:
        acc = O.merge_pair(acc, cores[j])
    return acc


def _subchain_block(prefix, last, c):
    """unfold_cyclic(subchain_skip(...), 1) restricted to lateral index i_{n-1} = c."""
    return O.unfold_cyclic(O.merge_pair(prefix, last[:, c:c + 1, :]), 1)


def mttsp(x, cores, n):
    """M_n = X_[n] @ G^{!=n}_[2] (solvers.py:375,379), blocked over i_{n-1}."""
    N = x.ndim
    if N < 3:
        return O.mttsp(x, cores, n)
    m = _slow_mode(n, N)
    pre = _prefix_chain(cores, n)
    out = None
    for c in range(x.shape[m]):
        part = _x_block_unfold(x, n, c) @ _subchain_block(pre, cores[m], c)
        out = part if out is None else out + part
    return out


def dense_slab(cores, c):
    """x_hat[..., c] of reconstruct(cores) (ring.py:155-170): the ring with the last core sliced."""
    cs = list(cores[:-1]) + [cores[-1][:, c:c + 1, :]]
    return O.dense_from_ring(cs, budget=1 << 62)[..., 0]


def residual_exact(x, cores):
    """solvers.py:164-174 blocked along the last mode."""
    nx = O.fro(x)
    if nx == 0.0:
        return 0.0
    acc = 0.0
    for c in range(x.shape[-1]):
        d = x[..., c] - dense_slab(cores, c)
        acc += float(np.dot(d.ravel(), d.ravel()))
    return math.sqrt(acc) / nx


def synth(recipe):
    """make_dataset (synthetic.py:184-197), gaussian kind, slab-wise reconstruct.

    Same streams as the reference: SeedSequence(seed).spawn(2) -> core stream,
    noise stream; the noise is one standard_normal draw of X's shape."""
    core_seq, noise_seq = O.child_seeds(recipe.seed, 2)
    rng = O.philox(core_seq)
    cores = [rng.standard_normal((recipe.rank, recipe.dim, recipe.rank)) for _ in range(recipe.order)]
    dims = (recipe.dim,) * recipe.order
    x = np.empty(dims, dtype=np.float64)
    for c in range(dims[-1]):
        x[..., c] = dense_slab(cores, c)
    if recipe.noise != 0.0:
        draw = O.philox(noise_seq).standard_normal(dims)
        scale = recipe.noise * (O.fro(x) / O.fro(draw))
        draw *= scale
        x += draw
        del draw
    return x, cores


def tsqr(blocks):
    """R (nonnegative diagonal) and the implicit Q of the row-stacked blocks (linalg.py:36-52).

    blocks: iterable of (rows_c x n) arrays.  Returns (r, qs, q2) with
    stack(blocks) = diag(qs) @ q2 @ r."""
    qs, rs = [], []
    for b in blocks:
        if b.shape[0] > b.shape[1]:
            q, r = np.linalg.qr(b, mode="reduced")
        else:
            q, r = None, b
        qs.append(q)
        rs.append(r)
    q2, r = np.linalg.qr(np.concatenate(rs, axis=0), mode="reduced")
    s = np.sign(np.diagonal(r)).copy()
    s[s == 0] = 1.0
    return r * s[:, None], qs, q2 * s


# ---------------------------------------------------------------------------
# the three sweeps (solvers.py:352-501) with the blocked products
# ---------------------------------------------------------------------------
class Run:
    """One solver run; `states[k]` = cores after sweep k (only the sweeps in `keep`)."""

    def __init__(self, x, variant, ranks, init, keep=()):
        self.x = x
        self.variant = variant
        self.N = x.ndim
        self.dims = x.shape
        self.ranks = list(ranks)
        self.cores = [np.array(g, dtype=np.float64, copy=True) for g in init]
        self.x_norm = O.fro(x)
        self.keep = set(keep)
        self.states = {}
        self.exact_errors, self.cheap_errors, self.fallbacks = [], [], 0
        if variant == "ne":
            self.grams = [O.bond_gram(g) for g in self.cores]
        else:
            self.qrs = [O.lateral_qr(g) for g in self.cores]
            if variant == "qrne":
                self.rgrams = [O.bond_gram(f.r_tensor) for f in self.qrs]

    def shape_of(self, n):
        return (self.ranks[n], self.dims[n], self.ranks[(n + 1) % self.N])

    def _normal(self, s, m):
        z, fb = O.solve_spd_right(s, m)
        self.fallbacks += int(fb)
        return z

    def _tri(self, r0, w):
        """solvers.py:262-273 with rank_deficient_fallback=True."""
        if r0.shape[0] != r0.shape[1]:
            return O.solve_pinv_right(r0, w)
        try:
            return O.solve_upper_right(r0, w)
        except O.DegenerateTriangularError:
            self.fallbacks += 1
            return O.solve_pinv_right(r0, w)

    def _y(self, n):
        y = O.mode_products(self.x, [(j, self.qrs[j].q.T) for j in range(self.N) if j != n])
        return np.ascontiguousarray(y)

    def block_ne(self, n):
        s = O.chain_grams(self.grams[j] for j in O.gram_order(n, self.N))
        m = mttsp(self.x, self.cores, n)
        z = self._normal(s, m)
        self.cores[n] = O.fold_classical(z, 1, self.shape_of(n))
        self.grams[n] = O.bond_gram(self.cores[n])
        return (float(np.vdot(m, z)), float(np.vdot(s, z.T @ z)))

    def block_qrne(self, n):
        N = self.N
        s = O.chain_grams(self.rgrams[j] for j in O.gram_order(n, N))
        y = self._y(n)
        rt = [f.r_tensor for f in self.qrs]
        m = None
        if N < 3:
            m = O.unfold_cyclic(y, n) @ O.unfold_cyclic(O.chain_without(rt, n), 1)
        else:
            sm = _slow_mode(n, N)
            pre = _prefix_chain(rt, n)
            for c in range(y.shape[sm]):
                part = _x_block_unfold(y, n, c) @ _subchain_block(pre, rt[sm], c)
                m = part if m is None else m + part
        del y
        z = self._normal(s, m)
        self.cores[n] = O.fold_classical(z, 1, self.shape_of(n))
        self.qrs[n] = O.lateral_qr(self.cores[n])
        self.rgrams[n] = O.bond_gram(self.qrs[n].r_tensor)
        rz = self.qrs[n].r_matrix
        return (float(np.vdot(m, z)), float(np.vdot(s, rz.T @ rz)))

    def block_qr(self, n):
        N = self.N
        rt = [f.r_tensor for f in self.qrs]
        y = self._y(n)
        sm = _slow_mode(n, N)
        rows = 1
        for j in range(N):
            if j != n:
                rows *= rt[j].shape[1]
        rr = self.ranks[n] * self.ranks[(n + 1) % N]
        if N < 3 or rows < rr:
            q0, r0 = O.qr_signed(O.unfold_cyclic(O.chain_without(rt, n), 1))
            w = O.unfold_cyclic(y, n) @ q0
        else:
            pre = _prefix_chain(rt, n)
            K = y.shape[sm]
            r0, qs, q2 = tsqr(_subchain_block(pre, rt[sm], c) for c in range(K))
            w = None
            off = 0
            for c in range(K):
                yc = _x_block_unfold(y, n, c)
                yq = yc @ qs[c] if qs[c] is not None else yc
                part = yq @ q2[off:off + yq.shape[1]]
                off += yq.shape[1]
                w = part if w is None else w + part
        del y
        z = self._tri(r0, w)
        self.cores[n] = O.fold_classical(z, 1, self.shape_of(n))
        self.qrs[n] = O.lateral_qr(self.cores[n])
        rz = self.qrs[n].r_matrix
        return (float(np.vdot(w, z @ r0.T)), float(np.vdot(r0.T @ r0, rz.T @ rz)))

    def sweep(self, exact=True):
        blk = {"ne": self.block_ne, "qr": self.block_qr, "qrne": self.block_qrne}[self.variant]
        terms = None
        for n in range(self.N):
            terms = blk(n)
        self.cheap_errors.append(O.residual_from_sweep(self.x_norm, *terms))
        if exact:
            self.exact_errors.append(residual_exact(self.x, self.cores))
        k = len(self.cheap_errors)
        if k in self.keep:
            self.states[k] = [g.copy() for g in self.cores]


def solve(x, variant, ranks, init, sweeps, keep=(), exact=True, log=None):
    """Run `sweeps` sweeps; returns the Run (errors, states, final cores)."""
    run = Run(x, variant, ranks, init, keep)
    for k in range(sweeps):
        run.sweep(exact=exact)
        if log is not None:
            log(k + 1, run)
    return run
