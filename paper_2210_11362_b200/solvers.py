"""Drop-in TR-ALS solvers (NE / QR / QRNE) running on the B200 engine.

Mirrors the reference's public surface for the north-star path
(pkg/src/tenring/solvers.py): `AlsConfig` (:60-104), `AlsReport`
(:107-133), `tr_als_ne` (:352-391), `tr_als_qr` (:403-451), `tr_als_qrne`
(:454-501) and `decompose` (:504-520), with the same arguments, defaults,
validation errors, zero-input rule, seeded initial cores (numpy Philox, the
exact draws of ring.random_cores) and returned objects.  The sweep itself
runs in `engine.SweepEngine` on the GPU; there is no CPU path.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from time import perf_counter

import numpy as np

from . import _lib as L
from .errors import DegenerateTriangularError, ElementBudgetError, StaleCacheError  # noqa: F401
from .host import (check_element_budget, check_ranks, core_ranks, make_rng,
                   random_cores, validate_cores, zero_cores)

VARIANTS = ("als", "ne", "qr", "qrne")          # solvers.py:55
DEVICE_VARIANTS = ("als", "ne", "qr", "qrne")
ERROR_MODES = ("exact", "cheap", "none")         # solvers.py:56
BUCKETS = ("subchain", "mttsp", "solve", "gramqr", "other")  # solvers.py:57
SVD_RCOND_DEFAULT = 1e-12                        # linalg.py:20
DTYPES = ("float64", "float32")                  # AlsConfig.dtype (extension)
FP64_GEMMS = ("auto", "ozaki", "crt", "dmma")            # AlsConfig.fp64_gemm (extension)


@dataclass
class AlsConfig:
    """Same fields and defaults as the reference AlsConfig (solvers.py:60-104).

    `shard_mode` (extension, 0-based) selects the mode X is split along when
    the call runs inside an initialised torch.distributed NCCL group (one
    process per GPU); it is ignored for single-process runs.  The default 0 is
    BASELINE's "mode 1" in the paper's 1-based numbering; with it every rank's
    slab is a contiguous block of X.

    `dtype` (extension) selects the storage/compute type of X's contractions:
    "float64" (default, the reference's) or "float32" -- the fp32 variant of
    BASELINE config 4: X is held in fp32 and the environment products run on
    the int8 tcgen05 tensor cores over 4 digit slices of X (exact int32
    accumulation), everything downstream in fp64; parity with the fp64
    reference is ~1e-4 instead of 1e-9.

    `fp64_gemm` (extension) selects the engine of the fp64 environment
    products (the X-streaming MTTSP, solvers.py:379): "dmma" runs them on the
    fp64 DMMA pipe; the int8 tcgen05 engine runs them with the accuracy of
    an fp64 product (measured against an extended-precision one) either as
    15 modular int8 GEMMs + an exact CRT reconstruction ("crt": contractions
    of K >= 4096 with R^2 <= 512) or as 28 exact digit-pair products over 7
    balanced digit slices ("ozaki").  "auto" (default) picks the int8 engine
    when 2 |X| R^2 >= 4 GFLOP (BASELINE c3-c5), per product the CRT form
    where it applies, provided the planes fit in free device memory and X
    passes the dynamic-range guard (include/trals.h).  X's
    planes (7 or 15 bytes per element and phase) are made once per call, timed as
    upfront_seconds["mttsp"].
    """

    ranks: tuple
    max_iters: int = 20
    tol: float = 0.0
    seed: object = None
    error_mode: str = "exact"
    rank_deficient_fallback: bool = True
    init_cores: list = None
    element_budget: int = None
    svd_rcond: float = SVD_RCOND_DEFAULT
    debug_checks: bool = False
    shard_mode: int = 0
    timing_buckets: bool = True
    dtype: str = "float64"
    fp64_gemm: str = "auto"


@dataclass
class AlsReport:
    """solvers.py:107-133; timings are CUDA-event device times."""

    variant: str
    errors: list = field(default_factory=list)
    iter_seconds: list = field(default_factory=list)
    iter_buckets: list = field(default_factory=list)
    upfront_seconds: dict = field(default_factory=dict)
    termination: str = ""
    fallback_count: int = 0

    @property
    def n_iters(self):
        return len(self.iter_seconds)

    @property
    def final_error(self):
        return self.errors[-1] if self.errors else None


@dataclass
class SweepCache:
    """End-of-sweep intermediates behind cheap_relative_error (reference solvers.py:140-161): same
    fields; only those of the variant are set, and `fresh` must be True (end of a full sweep)."""

    variant: str
    x_norm: float
    fresh: bool = False
    core_mat: np.ndarray = None      # updated last core, classical 2-unfolding
    m_last: np.ndarray = None        # als/ne/qrne: data-times-coefficient product
    s_last: np.ndarray = None        # ne/qrne: coefficient Gram matrix
    w_last: np.ndarray = None        # qr: compressed data block
    r0_last: np.ndarray = None       # qr: triangular factor of the subchain
    r_core_mat: np.ndarray = None    # qr/qrne: triangular factor of the updated core
    c_last: np.ndarray = None        # als: q.T @ X_cyc(n).T from the block QR
    r_a_last: np.ndarray = None      # als: triangular factor of the block QR


def cheap_relative_error(cache):
    """Relative error from sweep intermediates (reference solvers.py:177-212): sqrt(max(0, |X|^2 -
    2 cross + model)) / |X| with the variant's cross and model terms, evaluated on the GPU.  The solvers
    compute the same identity on the device every sweep (trals_error_terms_f64); this is the
    reference's standalone function for a caller-held cache."""
    import torch
    if not isinstance(cache, SweepCache):
        raise TypeError("cheap_relative_error expects a SweepCache")
    if not cache.fresh:
        raise StaleCacheError("cheap error is only defined at the end of a full sweep")
    if cache.x_norm == 0.0:
        return 0.0
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_11362_b200 needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())

    def t(a):
        return torch.as_tensor(np.asarray(a, dtype=np.float64), device=dev)

    def dot(a, b):
        return float(torch.sum(a * b).item())

    g = t(cache.core_mat)
    if cache.variant == "ne":
        cross, model = dot(t(cache.m_last), g), dot(t(cache.s_last), g.T @ g)
    elif cache.variant == "qr":
        r0, rz = t(cache.r0_last), t(cache.r_core_mat)
        cross, model = dot(t(cache.w_last), g @ r0.T), dot(r0.T @ r0, rz.T @ rz)
    elif cache.variant == "qrne":
        rz = t(cache.r_core_mat)
        cross, model = dot(t(cache.m_last), g), dot(t(cache.s_last), rz.T @ rz)
    elif cache.variant == "als":
        ra = t(cache.r_a_last)
        cross, model = dot(t(cache.c_last), ra @ g.T), dot(ra.T @ ra, g.T @ g)
    else:
        raise ValueError(f"unknown variant {cache.variant!r}")
    sq = cache.x_norm ** 2 - 2.0 * cross + model
    return math.sqrt(max(0.0, sq)) / cache.x_norm


def _validate(x, config, variant):
    """solvers.py:224-246 validation order and messages."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    if config.error_mode not in ERROR_MODES:
        raise ValueError(f"unknown error_mode {config.error_mode!r}; expected one of {ERROR_MODES}")
    if config.tol > 0 and config.error_mode == "none":
        raise ValueError("tol-based termination needs error tracking enabled")
    if config.max_iters < 1:
        raise ValueError("max_iters must be at least 1")
    if config.dtype not in DTYPES:
        raise ValueError(f"unknown dtype {config.dtype!r}; expected one of {DTYPES}")
    if config.fp64_gemm not in FP64_GEMMS:
        raise ValueError(f"unknown fp64_gemm {config.fp64_gemm!r}; expected one of {FP64_GEMMS}")


def _host_or_device_tensor(x, dtype="float64"):
    """Coerce the input like check_dense_tensor (validation.py:43-55) without a host pass over the data.

    Returns a torch tensor of `dtype` (host or device, possibly a view); the
    finite check runs later on the device (sumsq kernel)."""
    import torch
    td = torch.float64 if dtype == "float64" else torch.float32
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype != td:
            t = t.to(td)
    else:
        t = torch.from_numpy(np.asarray(x, dtype=np.float64 if dtype == "float64" else np.float32))
    if t.dim() < 2:
        raise ValueError(f"tensor order {t.dim()} is below the minimum 2")
    if t.numel() == 0:
        raise ValueError("tensor has no elements")
    return t


def _run(x, config, variant):
    import torch

    _validate(x, config, variant)
    t = _host_or_device_tensor(x, config.dtype)
    dims = tuple(int(d) for d in t.shape)
    N = len(dims)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_11362_b200 needs a CUDA device (no CPU fallback)")
    lib = L.lib()  # fail loudly if the extension is missing

    report = AlsReport(variant=variant)
    dist = _dist_context()
    dev = torch.device("cuda", torch.cuda.current_device())
    if dist is None:
        shard, lo, hi, world, group = None, 0, None, 1, None
        src = t
    else:
        world, rank, group = dist
        shard = int(config.shard_mode) % N
        lo, hi = _slab(dims[shard], world, rank)
        src = t.narrow(shard, lo, hi - lo)
    from .engine import OZ64_MAX_RHO, SweepEngine
    try:
        rk = tuple(int(r) for r in config.ranks)
    except (TypeError, ValueError):
        rk = None
    key = (dims, rk, variant, dev.index, world, shard, lo, hi, bool(config.rank_deficient_fallback),
           float(config.svd_rcond), config.dtype, bool(config.debug_checks), config.fp64_gemm)
    eng = _PLAN_CACHE.pop(key, None)
    x_local = eng.x if eng is not None else torch.empty(tuple(src.shape), dtype=t.dtype, device=dev)
    if src.is_cuda:
        x_local.copy_(src)
    else:
        if not src.is_contiguous():
            src = src.contiguous()
        x_local.copy_(src, non_blocking=bool(src.is_pinned()))
    # check_dense_tensor's finiteness test comes before the rank and budget checks
    # (solvers.py:235-242 -> validation.py:43-55); here it is one pass over X on the device
    xn_dev = _sumsq_device(lib, x_local, dev)
    if world > 1:
        import torch.distributed as tdist
        tdist.all_reduce(xn_dev, group=group)
    xn = xn_dev.cpu().numpy()
    if xn[1] > 0:
        if eng is not None:
            _PLAN_CACHE[key] = eng
        raise ValueError("tensor contains non-finite entries")  # validation.py:53-54
    ranks = check_ranks(config.ranks, N)
    if config.error_mode == "exact":
        check_element_budget(dims, config.element_budget)

    def build(gemm):
        return SweepEngine(x_local, dims, ranks, variant, shard_mode=shard, lo=lo, hi=hi, group=group,
                           world_size=world, rank_deficient_fallback=config.rank_deficient_fallback,
                           svd_rcond=config.svd_rcond, debug_checks=config.debug_checks, fp64_gemm=gemm)
    if eng is None:
        eng = build(config.fp64_gemm)
    if config.fp64_gemm == "auto":
        # accuracy guard of the int8 engine (include/trals.h): a row of X with a wide dynamic range
        # is held only to 2^-56.9 of its maximum, so such X runs on the fp64 DMMA pipe
        if eng.oz64:
            if _all_ranks_max(eng.x_dynamic_range(), world, group) > OZ64_MAX_RHO:
                eng = build("dmma")
                eng.guard_fallback = True
        elif getattr(eng, "guard_fallback", False):
            probe = build("auto")
            if probe.oz64 and _all_ranks_max(probe.x_dynamic_range(), world, group) <= OZ64_MAX_RHO:
                eng = probe
    eng.stream = torch.cuda.current_stream(dev)
    eng.xnorm2.copy_(xn_dev)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(eng.stream)
    eng.prepare_x()
    p1.record(eng.stream)
    if config.error_mode == "exact":
        eng.ensure_x64()
    _PLAN_CACHE[key] = eng
    while len(_PLAN_CACHE) > _PLAN_CACHE_MAX:
        _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
    xnorm2 = float(xn[0])
    if xnorm2 == 0.0:  # solvers.py:289-291
        report.termination = "zero_input"
        return zero_cores(dims, ranks), report

    # initial cores (solvers.py:248-257)
    if config.init_cores is not None:
        cores0 = validate_cores(config.init_cores, dims=dims)
        got = core_ranks(cores0)
        if got != tuple(ranks):
            raise ValueError(f"init cores have ranks {got}, expected {tuple(ranks)}")
        cores0 = [g.copy() for g in cores0]
    else:
        cores0 = random_cores(dims, ranks, make_rng(config.seed))

    stream = eng.stream
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    eng.set_cores(cores0)
    t1.record(stream)

    track = config.error_mode in ("exact", "cheap")
    exact = config.error_mode == "exact"
    use_graph = (not config.timing_buckets and not config.debug_checks and (world == 1 or _nccl(group)))
    if use_graph and (eng.graph is None or eng.graph_exact != exact):
        eng.capture(with_error=True, exact=exact)
    errs = torch.zeros((config.max_iters, 3), dtype=torch.float64, device=x_local.device)
    sweep_events = []
    report.termination = "max_iters"
    done = 0
    for k in range(config.max_iters):
        ev = [] if (config.timing_buckets and not use_graph) else None
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        # iter_seconds covers the sweep only; the error evaluation is excluded (solvers.py:111-116)
        if use_graph:
            eng.replay(sweep=True, error=False)
            b.record(stream)
            if track:
                eng.replay(sweep=False, error=True)
                errs[k].copy_(eng.err_cur)
        else:
            eng.run_sweep(ev)
            b.record(stream)
            if track:
                eng.error_step(errs[k], exact=exact)
        sweep_events.append((a, b, ev))
        done = k + 1
        if config.tol > 0 and k >= 1:
            e = errs[k - 1:k + 1, 0].cpu().numpy()
            if abs(e[0] - e[1]) < config.tol:
                report.termination = "tol"
                break
    torch.cuda.synchronize(x_local.device)
    _raise_on_info(eng, config, report)
    if variant != "als":  # tr_als has no prepare step (solvers.py:323-349)
        report.upfront_seconds["gramqr"] = t0.elapsed_time(t1) / 1e3
    if eng.sliced:  # X's digit planes for the tensor-core environment products (once per call)
        report.upfront_seconds["mttsp"] = p0.elapsed_time(p1) / 1e3
    for a, b, ev in sweep_events:
        report.iter_seconds.append(a.elapsed_time(b) / 1e3)
        buckets = dict.fromkeys(BUCKETS, 0.0)
        if ev:
            marks = ev + [(None, b)]
            for (bk, e0), (_, e1) in zip(marks[:-1], marks[1:]):
                buckets[bk] += e0.elapsed_time(e1) / 1e3
        report.iter_buckets.append(buckets)
    if track:
        report.errors = [float(v) for v in errs[:done, 0].cpu().numpy()]
    return eng.cores_host(), report


def _sumsq_device(lib, x, dev):
    """[sum x^2, #non-finite] of a device tensor (one deterministic pass, tensor_ops.py:237-239)."""
    import torch
    out = torch.empty(2, dtype=torch.float64, device=dev)
    ws = torch.empty(lib.trals_sumsq_ws_elems(), dtype=torch.float64, device=dev)
    fn = lib.trals_sumsq_f32 if x.dtype == torch.float32 else lib.trals_sumsq_f64
    L.check(fn(x.data_ptr(), x.numel(), out.data_ptr(), ws.data_ptr(),
               int(torch.cuda.current_stream(dev).cuda_stream)), "sumsq")
    return out


def _all_ranks_max(v, world, group):
    """The same engine choice on every rank: the guard statistic max-reduced over the ranks."""
    if world <= 1:
        return v
    import torch
    import torch.distributed as tdist
    t = torch.tensor([v], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX, group=group)
    return float(t.item())


def _nccl(group):
    import torch.distributed as tdist
    return tdist.get_backend(group) == "nccl"


_PLAN_CACHE = {}
_PLAN_CACHE_MAX = 2


def clear_plan_cache():
    """Drop cached engines (device buffers, captured graphs)."""
    _PLAN_CACHE.clear()


def _raise_on_info(eng, config, report):
    info = eng.info.cpu().numpy().copy()
    eng.info.zero_()
    report.fallback_count = int(info[L.INFO_FALLBACKS])  # solvers.py:262-279
    if info[L.INFO_ASYM]:
        raise ValueError("matrix is not symmetric within 1e-8 relative")  # linalg.py:70-72
    if info[L.INFO_DEGEN] or (config is not None and eng.variant in ("qr", "als") and info[L.INFO_CHOL]):
        # only left set when rank_deficient_fallback is off (linalg.py:96-99, solvers.py:269-270)
        idx = int(info[L.INFO_DEGEN] or info[L.INFO_CHOL]) - 1
        raise DegenerateTriangularError(idx, 0.0, 0.0)
    if info[L.INFO_CHOL]:
        raise np.linalg.LinAlgError(f"Cholesky failed at pivot {int(info[L.INFO_CHOL])}")


def _dist_context():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return None
    if not (dist.is_available() and dist.is_initialized()):
        return None
    world = dist.get_world_size()
    if world <= 1:
        return None
    return world, dist.get_rank(), None


def _slab(I, world, rank):
    base, extra = divmod(I, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def tr_als_ne(x, config):
    """Normal-equation sweep (Alg. 2; reference solvers.py:352-391). Returns (cores, report)."""
    return _run(x, config, "ne")


def tr_als_qr(x, config):
    """QR-stabilised sweep (Alg. 3; reference solvers.py:403-451). Returns (cores, report)."""
    return _run(x, config, "qr")


def tr_als_qrne(x, config):
    """Compressed NE sweep (Alg. 4; reference solvers.py:454-501). Returns (cores, report)."""
    return _run(x, config, "qrne")


def tr_als(x, config):
    """Plain TR-ALS (Alg. 1; reference solvers.py:323-349). Returns (cores, report).

    The reference materialises each subchain unfolding A_n (prod_{j!=n} I_j x R^2)
    and solves by its QR.  Here A_n is never formed: the right-hand side is the
    same environment-tree MTTSP as NE, and R is the nonnegative-diagonal Cholesky
    factor of S_n = A_n^T A_n -- the same R in exact arithmetic -- with the
    reference's triangular-solve policy (degeneracy floor, counted SVD fallback,
    uncounted min-norm solve when A_n has fewer rows than R^2, solvers.py:262-273)."""
    return _run(x, config, "als")


_SOLVERS = {"als": tr_als, "ne": tr_als_ne, "qr": tr_als_qr, "qrne": tr_als_qrne}


def decompose(x, variant, config):
    """Run the named solver variant (reference solvers.py:504-520)."""
    try:
        solver = _SOLVERS[variant]
    except KeyError:
        raise ValueError(f"unknown variant {variant!r}; expected one of {VARIANTS}") from None
    return solver(x, config)
