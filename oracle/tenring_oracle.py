"""CPU oracle for the TR-ALS hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package `tenring`
0.1.0 (pkg/src/tenring under the upstream reference tree) for exactly the
functions on the north-star path: the NE, QR and QRNE sweeps, their run
scaffolding (validation, seeded initialisation, termination, error
tracking), the ring algebra they call, and the synthetic-data recipe used to
build their inputs.  Every function cites the reference file:line it
follows.

Who may use it: `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline`
/ `--impl reference` legs of `bench.py` -- as the checker or as the timed
CPU stand-in for the reference, never as the product.  The product package
(`paper_2210_11362_b200`) must not import this module.

Parity pin: the restatement is checked against golden vectors produced by
running the real reference in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`), see
`tests/test_oracle_golden.py`.

Operation order deliberately mirrors the reference (materialised subchain,
cyclic-unfold copies, numpy/LAPACK calls) so that timing this module on the
GPU host is a faithful CPU baseline of the reference's path.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from time import perf_counter

import numpy as np
import scipy.linalg as sla

# ---------------------------------------------------------------------------
# validation.py:8-73
# ---------------------------------------------------------------------------
BUDGET_DEFAULT = 1 << 27  # validation.py:8
BUDGET_ENV = "TENRING_BUDGET"  # validation.py:9


class ElementBudgetError(MemoryError):
    """validation.py:12-14."""


def resolve_budget(override=None):
    """validation.py:17-28: explicit > env var > 2**27."""
    if override is not None:
        return int(override)
    env = os.environ.get(BUDGET_ENV)
    return int(env) if env is not None else BUDGET_DEFAULT


def guard_budget(shape, budget=None):
    """validation.py:31-40."""
    count = math.prod(int(d) for d in shape)
    cap = resolve_budget(budget)
    if count > cap:
        raise ElementBudgetError(
            f"dense tensor with {count} elements exceeds the element budget of {cap}")
    return count


def as_dense(x, min_order=1):
    """validation.py:43-55: float64 coercion, order, nonempty, finite."""
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim < min_order:
        raise ValueError(f"tensor order {arr.ndim} is below the minimum {min_order}")
    if arr.size == 0:
        raise ValueError("tensor has no elements")
    if not np.isfinite(arr).all():
        raise ValueError("tensor contains non-finite entries")
    return arr


def as_ranks(ranks, order):
    """validation.py:58-65."""
    out = [int(r) for r in ranks]
    if len(out) != order:
        raise ValueError(f"expected {order} ranks, got {len(out)}")
    if min(out) < 1:
        raise ValueError("ranks must be positive")
    return out


# ---------------------------------------------------------------------------
# utils.py:9-32 -- Philox4x32 over SeedSequence
# ---------------------------------------------------------------------------
def philox(seed=None):
    """utils.py:9-23."""
    if isinstance(seed, np.random.Generator):
        return seed
    seq = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    return np.random.Generator(np.random.Philox(seq))


def child_seeds(seed, count):
    """utils.py:26-32."""
    seq = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    return seq.spawn(count)


# ---------------------------------------------------------------------------
# tensor_ops.py -- unfoldings are first-index-fastest (Fortran) linearisations
# ---------------------------------------------------------------------------
def _perm_cyclic(n, order):
    # tensor_ops.py:44-45: rows = mode n, columns = n+1..N-1, 0..n-1
    return [n, *range(n + 1, order), *range(n)]


def _perm_classical(n, order):
    # tensor_ops.py:48-49: rows = mode n, columns = remaining modes ascending
    return [n, *(j for j in range(order) if j != n)]


def _detach(view, base):
    # tensor_ops.py:37-41: results never alias their input.  The copy keeps
    # numpy's default (C) order so BLAS sees the same operand layouts.
    return view.copy() if np.shares_memory(view, base) else view


def unfold_cyclic(x, n):
    """tensor_ops.py:69-81."""
    x = np.asarray(x)
    return _detach(x.transpose(_perm_cyclic(n, x.ndim)).reshape(x.shape[n], -1, order="F"), x)


def unfold_classical(x, n):
    """tensor_ops.py:52-66."""
    x = np.asarray(x)
    return _detach(x.transpose(_perm_classical(n, x.ndim)).reshape(x.shape[n], -1, order="F"), x)


def unfold_split(x, k):
    """tensor_ops.py:84-97."""
    x = np.asarray(x)
    rows = int(np.prod(x.shape[:k])) if k else 1
    return _detach(x.reshape(rows, -1, order="F"), x)


def fold_classical(m, n, shape):
    """tensor_ops.py:100-108."""
    m = np.asarray(m)
    perm = _perm_classical(n, len(shape))
    t = m.reshape([shape[j] for j in perm], order="F")
    return _detach(t.transpose(np.argsort(perm)), m)


def fold_cyclic(m, n, shape):
    """tensor_ops.py:111-119."""
    m = np.asarray(m)
    perm = _perm_cyclic(n, len(shape))
    t = m.reshape([shape[j] for j in perm], order="F")
    return _detach(t.transpose(np.argsort(perm)), m)


def mode_product(x, u, n):
    """tensor_ops.py:145-162: out[..., j, ...] = sum_i u[j, i] x[..., i, ...]."""
    return np.moveaxis(np.tensordot(u, x, axes=(1, n)), 0, n)


def mode_products(x, pairs):
    """tensor_ops.py:165-181 (ascending mode order)."""
    out = np.asarray(x)
    for n, u in sorted(pairs, key=lambda p: p[0]):
        out = mode_product(out, u, n)
    return out


def compose_grams(a, b):
    """tensor_ops.py:206-225: out[i,j,r,s] = sum_{m,k} a[i,m,r,k] b[m,j,k,s]."""
    return np.einsum("imrk,mjks->ijrs", a, b, optimize=True)


def fro(a):
    """tensor_ops.py:237-239."""
    return float(np.linalg.norm(np.asarray(a).ravel()))


# ---------------------------------------------------------------------------
# linalg.py:36-112
# ---------------------------------------------------------------------------
TRI_FLOOR = 1e-13  # linalg.py:19
SVD_RCOND = 1e-12  # linalg.py:20


class DegenerateTriangularError(np.linalg.LinAlgError):
    """linalg.py:23-33."""

    def __init__(self, index, value, floor):
        self.index, self.value, self.floor = int(index), float(value), float(floor)
        super().__init__(f"triangular factor diagonal {value:.3e} at index {index} "
                         f"is below the degeneracy floor {floor:.3e}")


def qr_signed(a):
    """linalg.py:36-52: economy QR with nonnegative diag(R)."""
    q, r = np.linalg.qr(np.asarray(a, dtype=np.float64), mode="reduced")
    s = np.sign(np.diagonal(r)).copy()
    s[s == 0] = 1.0
    return q * s, r * s[:, None]


def solve_spd_right(s, rhs):
    """linalg.py:55-81: z @ s = rhs by upper Cholesky; gelsy LS fallback.

    Returns (z, used_fallback)."""
    s = np.asarray(s, dtype=np.float64)
    rhs = np.asarray(rhs, dtype=np.float64)
    scale = np.max(np.abs(s)) if s.size else 0.0
    if scale > 0 and np.max(np.abs(s - s.T)) > 1e-8 * scale:
        raise ValueError("matrix is not symmetric within 1e-8 relative")
    sym = 0.5 * (s + s.T)
    try:
        factor = sla.cho_factor(sym, lower=False, check_finite=False)
        return sla.cho_solve(factor, rhs.T, check_finite=False).T, False
    except (sla.LinAlgError, np.linalg.LinAlgError):
        z = sla.lstsq(sym, rhs.T, lapack_driver="gelsy", check_finite=False)[0]
        return z.T, True


def solve_upper_right(r, rhs, floor_scale=TRI_FLOOR):
    """linalg.py:84-101: z @ r.T = rhs with the 1e-13 degeneracy floor."""
    r = np.asarray(r, dtype=np.float64)
    d = np.abs(np.diagonal(r))
    floor = floor_scale * (np.max(np.abs(r)) if r.size else 0.0)
    k = int(np.argmin(d))
    if d[k] <= floor:
        raise DegenerateTriangularError(k, d[k], floor)
    return sla.solve_triangular(r, np.asarray(rhs, dtype=np.float64).T, lower=False,
                                check_finite=False).T


def solve_pinv_right(r, rhs, rcond=SVD_RCOND):
    """linalg.py:104-112."""
    return np.asarray(rhs, dtype=np.float64) @ np.linalg.pinv(np.asarray(r, dtype=np.float64),
                                                              rcond=rcond).T


# ---------------------------------------------------------------------------
# ring.py -- cores are (R_n, I_n, R_{n+1})
# ---------------------------------------------------------------------------
def check_cores(cores, dims=None):
    """ring.py:62-84."""
    cs = [np.asarray(g, dtype=np.float64) for g in cores]
    if not cs:
        raise ValueError("a ring needs at least one core")
    for n, g in enumerate(cs):
        if g.ndim != 3:
            raise ValueError(f"core {n} has order {g.ndim}, expected 3")
        if g.shape[2] != cs[(n + 1) % len(cs)].shape[0]:
            raise ValueError(f"bond mismatch between core {n} and core {(n + 1) % len(cs)}")
    if dims is not None and tuple(g.shape[1] for g in cs) != tuple(dims):
        raise ValueError("core lateral sizes do not match dims")
    return cs


def bond_dims(cores):
    """ring.py:87-89."""
    return tuple(g.shape[0] for g in cores)


def gaussian_ring(dims, ranks, rng):
    """ring.py:92-98: N(0,1) cores drawn for n = 0..N-1 in C order."""
    N = len(dims)
    return [rng.standard_normal((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


def zero_ring(dims, ranks):
    """ring.py:101-107."""
    N = len(dims)
    return [np.zeros((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


def merge_pair(a, b):
    """ring.py:110-131: slice (j1 + J1*j2) = a[:, j1, :] @ b[:, j2, :]."""
    ia, ja, k = a.shape
    _, jb, ib = b.shape
    prod = (a.reshape(ia * ja, k) @ b.reshape(k, jb * ib)).reshape(ia, ja, jb, ib)
    return np.ascontiguousarray(prod.transpose(0, 2, 1, 3)).reshape(ia, jb * ja, ib)


def ring_order_without(n, N):
    """ring.py:134-135."""
    return [*range(n + 1, N), *range(n)]


def chain_without(cores, n):
    """ring.py:138-152: subchain tensor (R_{n+1}, prod_{j!=n} I_j, R_n)."""
    order = ring_order_without(n, len(cores))
    acc = cores[order[0]]
    for j in order[1:]:
        acc = merge_pair(acc, cores[j])
    return acc


def dense_from_ring(cores, budget=None):
    """ring.py:155-170."""
    cores = check_cores(cores)
    dims = tuple(g.shape[1] for g in cores)
    guard_budget(dims, budget)
    rest = chain_without(cores, 0)
    return fold_cyclic(unfold_classical(cores[0], 1) @ unfold_cyclic(rest, 1).T, 0, dims)


def bond_gram(g, z=None):
    """ring.py:173-188: P[a,b,c,d] = sum_i g[b,i,a] z[d,i,c]."""
    z = g if z is None else z
    return np.einsum("bia,dic->abcd", g, z, optimize=True)


def gram_order(n, N):
    """ring.py:191-198: n-1..0, N-1..n+1."""
    return [*range(n - 1, -1, -1), *range(N - 1, n, -1)]


def chain_grams(grams):
    """ring.py:201-214 -> R_nR_{n+1} square matrix, left bond fastest."""
    grams = list(grams)
    acc = grams[0]
    for p in grams[1:]:
        acc = compose_grams(acc, p)
    return unfold_split(acc, 2)


@dataclass
class LateralQr:
    """ring.py:217-233."""
    r_tensor: np.ndarray
    q: np.ndarray

    @property
    def r_matrix(self):
        return unfold_classical(self.r_tensor, 1)


def lateral_qr(g):
    """ring.py:236-249."""
    g = np.asarray(g, dtype=np.float64)
    q, r = qr_signed(unfold_classical(g, 1))
    return LateralQr(r_tensor=fold_classical(r, 1, (g.shape[0], r.shape[0], g.shape[2])), q=q)


# ---------------------------------------------------------------------------
# synthetic.py:39-197 (gaussian recipe used by BASELINE configs)
# ---------------------------------------------------------------------------
@dataclass
class Recipe:
    """synthetic.py:39-81 (gaussian / congruent / student_t fields)."""
    order: int = 3
    dim: int = 100
    rank: int = 5
    kind: str = "gaussian"
    noise: float = 0.0
    gamma: float = 0.5
    theta: float = 0.5
    dof: int = 1
    seed: object = None


def noisy(x_true, eta, rng):
    """synthetic.py:167-181: x + eta*||x||/||n|| * n."""
    if eta == 0.0:
        return x_true
    draw = rng.standard_normal(x_true.shape)
    return x_true + eta * (fro(x_true) / fro(draw)) * draw


def synth(recipe, budget=None):
    """synthetic.py:184-197 for kind='gaussian' (synthetic.py:84-91)."""
    if recipe.kind != "gaussian":
        raise NotImplementedError("oracle restates the gaussian recipe only")
    guard_budget([recipe.dim] * recipe.order, budget)
    core_seq, noise_seq = child_seeds(recipe.seed, 2)
    rng = philox(core_seq)
    cores = [rng.standard_normal((recipe.rank, recipe.dim, recipe.rank)) for _ in range(recipe.order)]
    x = noisy(dense_from_ring(cores, budget=budget), recipe.noise, philox(noise_seq))
    return x, cores


# ---------------------------------------------------------------------------
# solvers.py -- configuration, report, scaffolding and the three sweeps
# ---------------------------------------------------------------------------
VARIANTS = ("als", "ne", "qr", "qrne")  # solvers.py:55
ERROR_MODES = ("exact", "cheap", "none")  # solvers.py:56
BUCKETS = ("subchain", "mttsp", "solve", "gramqr", "other")  # solvers.py:57


@dataclass
class Config:
    """solvers.py:60-104 (same fields and defaults as AlsConfig)."""
    ranks: tuple
    max_iters: int = 20
    tol: float = 0.0
    seed: object = None
    error_mode: str = "exact"
    rank_deficient_fallback: bool = True
    init_cores: list = None
    element_budget: int = None
    svd_rcond: float = SVD_RCOND
    debug_checks: bool = False


@dataclass
class Report:
    """solvers.py:107-133."""
    variant: str
    errors: list = field(default_factory=list)
    iter_seconds: list = field(default_factory=list)
    iter_buckets: list = field(default_factory=list)
    upfront_seconds: dict = field(default_factory=dict)
    termination: str = ""
    fallback_count: int = 0


class _Clock:
    def __init__(self, buckets, key):
        self.buckets, self.key = buckets, key

    def __enter__(self):
        self.t = perf_counter()

    def __exit__(self, *exc):
        self.buckets[self.key] += perf_counter() - self.t


def residual_exact(x, cores, budget=None):
    """solvers.py:164-174."""
    nx = fro(x)
    return 0.0 if nx == 0.0 else fro(x - dense_from_ring(cores, budget=budget)) / nx


def residual_from_sweep(x_norm, cross, model):
    """solvers.py:207-212 (after the per-variant cross/model terms :194-205)."""
    if x_norm == 0.0:
        return 0.0
    return math.sqrt(max(0.0, x_norm ** 2 - 2.0 * cross + model)) / x_norm


class _Driver:
    """solvers.py:221-320."""

    def __init__(self, x, cfg, variant):
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r}")
        if cfg.error_mode not in ERROR_MODES:
            raise ValueError(f"unknown error_mode {cfg.error_mode!r}")
        if cfg.tol > 0 and cfg.error_mode == "none":
            raise ValueError("tol-based termination needs error tracking enabled")
        if cfg.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        self.x = as_dense(x, min_order=2)
        self.cfg, self.variant = cfg, variant
        self.dims, self.N = self.x.shape, self.x.ndim
        self.ranks = as_ranks(cfg.ranks, self.N)
        if cfg.error_mode == "exact":
            guard_budget(self.dims, cfg.element_budget)
        self.x_norm = fro(self.x)
        self.report = Report(variant=variant)
        self.last = {}
        self.buckets = None

    def shape_of(self, n):
        return (self.ranks[n], self.dims[n], self.ranks[(n + 1) % self.N])

    def start_cores(self):
        """solvers.py:248-257."""
        if self.cfg.init_cores is not None:
            cs = check_cores(self.cfg.init_cores, dims=self.dims)
            if bond_dims(cs) != tuple(self.ranks):
                raise ValueError(f"init cores have ranks {bond_dims(cs)}, expected {tuple(self.ranks)}")
            return [g.copy() for g in cs]
        return gaussian_ring(self.dims, self.ranks, philox(self.cfg.seed))

    def tri_block(self, r, rhs):
        """solvers.py:262-273."""
        if r.shape[0] != r.shape[1]:
            return solve_pinv_right(r, rhs, rcond=self.cfg.svd_rcond)
        try:
            return solve_upper_right(r, rhs)
        except DegenerateTriangularError:
            if not self.cfg.rank_deficient_fallback:
                raise
            self.report.fallback_count += 1
            return solve_pinv_right(r, rhs, rcond=self.cfg.svd_rcond)

    def normal_block(self, s, rhs):
        """solvers.py:275-279."""
        z, fb = solve_spd_right(s, rhs)
        self.report.fallback_count += int(fb)
        return z

    def run(self, sweep, prepare=None):
        """solvers.py:281-315."""
        rep = self.report
        if self.x_norm == 0.0:
            rep.termination = "zero_input"
            return zero_ring(self.dims, self.ranks), rep
        cores = self.start_cores()
        if prepare is not None:
            t0 = perf_counter()
            prepare(cores)
            rep.upfront_seconds["gramqr"] = rep.upfront_seconds.get("gramqr", 0.0) + perf_counter() - t0
        rep.termination = "max_iters"
        for _ in range(self.cfg.max_iters):
            self.buckets = dict.fromkeys(BUCKETS, 0.0)
            t0 = perf_counter()
            sweep(cores)
            rep.iter_seconds.append(perf_counter() - t0)
            rep.iter_buckets.append(self.buckets)
            if self.cfg.error_mode == "exact":
                rep.errors.append(residual_exact(self.x, cores, budget=self.cfg.element_budget))
            elif self.cfg.error_mode == "cheap":
                rep.errors.append(residual_from_sweep(self.x_norm, *self.last["terms"]))
            if self.cfg.tol > 0 and len(rep.errors) >= 2 and abs(rep.errors[-2] - rep.errors[-1]) < self.cfg.tol:
                rep.termination = "tol"
                break
        return cores, rep


def als_ne(x, cfg):
    """solvers.py:352-391 (Alg. 2, TR-ALS-NE)."""
    d = _Driver(x, cfg, "ne")
    if d.x_norm == 0.0:
        return d.run(None)
    xs = [unfold_cyclic(d.x, n) for n in range(d.N)]  # solvers.py:362
    grams = []

    def prepare(cores):
        grams.extend(bond_gram(g) for g in cores)

    def sweep(cores):
        for n in range(d.N):
            with _Clock(d.buckets, "other"):
                s = chain_grams(grams[j] for j in gram_order(n, d.N))
            with _Clock(d.buckets, "subchain"):
                a = unfold_cyclic(chain_without(cores, n), 1)
            with _Clock(d.buckets, "mttsp"):
                m = xs[n] @ a  # solvers.py:379, the MTTSP
            with _Clock(d.buckets, "solve"):
                z = d.normal_block(s, m)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
            with _Clock(d.buckets, "gramqr"):
                grams[n] = bond_gram(cores[n])
        # solvers.py:195-197 cheap-error terms from the last block
        d.last["terms"] = (float(np.vdot(m, z)), float(np.vdot(s, z.T @ z)))
        d.last["m"], d.last["s"], d.last["z"] = m, s, z

    return d.run(sweep, prepare)


def als_qr(x, cfg):
    """solvers.py:403-451 (Alg. 3, TR-ALS-QR)."""
    d = _Driver(x, cfg, "qr")
    if d.x_norm == 0.0:
        return d.run(None)
    qrs = []

    def prepare(cores):
        qrs.extend(lateral_qr(g) for g in cores)

    def sweep(cores):
        for n in range(d.N):
            with _Clock(d.buckets, "subchain"):
                v = chain_without([f.r_tensor for f in qrs], n)
            with _Clock(d.buckets, "gramqr"):
                q0, r0 = qr_signed(unfold_cyclic(v, 1))
            with _Clock(d.buckets, "mttsp"):
                y = mode_products(d.x, [(j, qrs[j].q.T) for j in range(d.N) if j != n])
            with _Clock(d.buckets, "other"):
                w = unfold_cyclic(y, n) @ q0
            with _Clock(d.buckets, "solve"):
                z = d.tri_block(r0, w)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
            with _Clock(d.buckets, "gramqr"):
                qrs[n] = lateral_qr(cores[n])
        rz = qrs[-1].r_matrix
        # solvers.py:198-201
        d.last["terms"] = (float(np.vdot(w, z @ r0.T)), float(np.vdot(r0.T @ r0, rz.T @ rz)))
        d.last["w"], d.last["r0"], d.last["z"] = w, r0, z

    return d.run(sweep, prepare)


def als_qrne(x, cfg):
    """solvers.py:454-501 (Alg. 4, TR-ALS-QRNE)."""
    d = _Driver(x, cfg, "qrne")
    if d.x_norm == 0.0:
        return d.run(None)
    qrs, rgrams = [], []

    def prepare(cores):
        qrs.extend(lateral_qr(g) for g in cores)
        rgrams.extend(bond_gram(f.r_tensor) for f in qrs)

    def sweep(cores):
        for n in range(d.N):
            with _Clock(d.buckets, "other"):
                s = chain_grams(rgrams[j] for j in gram_order(n, d.N))
            with _Clock(d.buckets, "subchain"):
                v = chain_without([f.r_tensor for f in qrs], n)
            with _Clock(d.buckets, "mttsp"):
                y = mode_products(d.x, [(j, qrs[j].q.T) for j in range(d.N) if j != n])
                m = unfold_cyclic(y, n) @ unfold_cyclic(v, 1)
            with _Clock(d.buckets, "solve"):
                z = d.normal_block(s, m)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
            with _Clock(d.buckets, "gramqr"):
                qrs[n] = lateral_qr(cores[n])
                rgrams[n] = bond_gram(qrs[n].r_tensor)
        rz = qrs[-1].r_matrix
        # solvers.py:202-205
        d.last["terms"] = (float(np.vdot(m, z)), float(np.vdot(s, rz.T @ rz)))
        d.last["m"], d.last["s"], d.last["z"] = m, s, z

    return d.run(sweep, prepare)


def als_plain(x, cfg):
    """solvers.py:323-349 (Alg. 1, TR-ALS): explicit subchain, QR least squares per block."""
    d = _Driver(x, cfg, "als")
    if d.x_norm == 0.0:
        return d.run(None)
    xs = [unfold_cyclic(d.x, n) for n in range(d.N)]  # solvers.py:331

    def sweep(cores):
        for n in range(d.N):
            with _Clock(d.buckets, "subchain"):
                a = unfold_cyclic(chain_without(cores, n), 1)
            with _Clock(d.buckets, "solve"):
                q, r = qr_signed(a)
                c = q.T @ xs[n].T
                z = d.tri_block(r, c.T)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
        # solvers.py:199-200 (c_last, r_a_last, core_mat of the last block)
        d.last["terms"] = (float(np.vdot(c, r @ z.T)), float(np.vdot(r.T @ r, z.T @ z)))
        d.last["c"], d.last["r"], d.last["z"] = c, r, z

    return d.run(sweep)


SOLVERS = {"als": als_plain, "ne": als_ne, "qr": als_qr, "qrne": als_qrne}


def solve(x, variant, cfg):
    """solvers.py:504-520."""
    if variant not in SOLVERS:
        raise ValueError(f"unknown variant {variant!r}")
    return SOLVERS[variant](x, cfg)


# ---------------------------------------------------------------------------
# direct building blocks used by the kernel-level parity tests
# ---------------------------------------------------------------------------
def mttsp(x, cores, n):
    """M_n = X_[n] @ G^{!=n}_[2] (solvers.py:375,379): I_n x R_n R_{n+1}."""
    return unfold_cyclic(x, n) @ unfold_cyclic(chain_without(cores, n), 1)


def coefficient_gram(cores, n):
    """S_n via the Gram chain (solvers.py:372-373, Prop. 3)."""
    return chain_grams(bond_gram(cores[j]) for j in gram_order(n, len(cores)))


class BlockStepper:
    """The reference's sweep body, one block update per call (CPU baseline legs of bench.py).

    `prepare()` does the untimed set-up of the reference's run (the N cyclic
    unfoldings of X, solvers.py:362; the initial Grams / lateral QRs,
    solvers.py:366-367, :417, :468-470); `step(n)` is exactly one iteration
    n of the per-mode loop of tr_als_ne (solvers.py:370-384), tr_als_qr
    (:420-443) or tr_als_qrne (:473-493), with the same materialised subchain,
    unfold copies and numpy/LAPACK calls as the functions above."""

    def __init__(self, x, variant, ranks, init):
        if variant not in ("ne", "qr", "qrne"):
            raise ValueError(f"unsupported variant {variant!r}")
        self.d = _Driver(x, Config(ranks=tuple(ranks), max_iters=1, init_cores=init, error_mode="none"), variant)
        self.variant = variant
        self.cores = self.d.start_cores()
        self.d.buckets = dict.fromkeys(BUCKETS, 0.0)

    def prepare(self):
        d = self.d
        if self.variant == "ne":
            self.xs = [unfold_cyclic(d.x, n) for n in range(d.N)]
            self.grams = [bond_gram(g) for g in self.cores]
        else:
            self.qrs = [lateral_qr(g) for g in self.cores]
            if self.variant == "qrne":
                self.rgrams = [bond_gram(f.r_tensor) for f in self.qrs]

    def step(self, n):
        d, cores = self.d, self.cores
        if self.variant == "ne":
            s = chain_grams(self.grams[j] for j in gram_order(n, d.N))
            a = unfold_cyclic(chain_without(cores, n), 1)
            m = self.xs[n] @ a
            del a
            z = d.normal_block(s, m)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
            self.grams[n] = bond_gram(cores[n])
        elif self.variant == "qr":
            v = chain_without([f.r_tensor for f in self.qrs], n)
            q0, r0 = qr_signed(unfold_cyclic(v, 1))
            del v
            y = mode_products(d.x, [(j, self.qrs[j].q.T) for j in range(d.N) if j != n])
            w = unfold_cyclic(y, n) @ q0
            del y, q0
            z = d.tri_block(r0, w)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
            self.qrs[n] = lateral_qr(cores[n])
        else:
            s = chain_grams(self.rgrams[j] for j in gram_order(n, d.N))
            v = chain_without([f.r_tensor for f in self.qrs], n)
            y = mode_products(d.x, [(j, self.qrs[j].q.T) for j in range(d.N) if j != n])
            m = unfold_cyclic(y, n) @ unfold_cyclic(v, 1)
            del y, v
            z = d.normal_block(s, m)
            cores[n] = fold_classical(z, 1, d.shape_of(n))
            self.qrs[n] = lateral_qr(cores[n])
            self.rgrams[n] = bond_gram(self.qrs[n].r_tensor)
