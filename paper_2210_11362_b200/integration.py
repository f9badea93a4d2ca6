"""Route a `tenring` installation's solver entry points to the B200 drop-in.

The reference's front ends reach the hot path only through `tenring.solvers`:
`TensorRingALS.fit` calls `decompose` (estimator.py:10, :107), `tenring decompose`
calls it (cli.py:16, :65), `bench.trial_rows` too (bench.py:175).  `install()`
rebinds those names -- the `_SOLVERS` table and `decompose` in `tenring.solvers`,
the `tr_als*` / `decompose` names re-exported by the package, and the copies the
estimator and CLI modules imported -- to wrappers that convert the reference's
`AlsConfig` into this package's (same fields), run the GPU solver, and hand the
result back as the reference's own `AlsReport`.  `uninstall()` restores the
originals.  This is the maintainer's one-line switch described in INTEGRATION.md:

    import tenring
    from paper_2210_11362_b200 import integration
    integration.install(tenring)          # every front end now runs on the GPU
"""

from __future__ import annotations

import dataclasses

from . import solvers as _ours

_FIELDS = ("ranks", "max_iters", "tol", "seed", "error_mode", "rank_deficient_fallback", "init_cores",
           "element_budget", "svd_rcond", "debug_checks")
_SAVED = {}


def _convert_config(cfg):
    """Reference AlsConfig (solvers.py:60-104) -> ours, field by field."""
    if isinstance(cfg, _ours.AlsConfig):
        return cfg
    return _ours.AlsConfig(**{f: getattr(cfg, f) for f in _FIELDS})


def _wrap(variant, ref_solvers):
    def solver(x, config):
        cores, rep = _ours._run(x, _convert_config(config), variant)
        out = ref_solvers.AlsReport(variant=rep.variant)
        for f in dataclasses.fields(out):
            setattr(out, f.name, getattr(rep, f.name))
        return cores, out
    solver.__name__ = f"tr_als_{variant}" if variant != "als" else "tr_als"
    solver.__doc__ = f"B200 drop-in for tenring.solvers.{solver.__name__} (paper_2210_11362_b200)."
    return solver


def install(tenring):
    """Rebind the reference package's solver entry points (see module docstring); idempotent."""
    import importlib
    rs = importlib.import_module(tenring.__name__ + ".solvers")
    est = importlib.import_module(tenring.__name__ + ".estimator")
    cli = importlib.import_module(tenring.__name__ + ".cli")
    if _SAVED:
        return
    wrapped = {v: _wrap(v, rs) for v in ("als", "ne", "qr", "qrne")}

    def decompose(x, variant, config):
        try:
            solver = wrapped[variant]
        except KeyError:
            raise ValueError(f"unknown variant {variant!r}; expected one of {rs.VARIANTS}") from None
        return solver(x, config)

    names = {"tr_als": wrapped["als"], "tr_als_ne": wrapped["ne"], "tr_als_qr": wrapped["qr"],
             "tr_als_qrne": wrapped["qrne"], "decompose": decompose}
    _SAVED["solvers"] = {n: getattr(rs, n) for n in names}
    _SAVED["solvers"]["_SOLVERS"] = dict(rs._SOLVERS)
    _SAVED["package"] = {n: getattr(tenring, n) for n in names if hasattr(tenring, n)}
    _SAVED["estimator"] = est.decompose
    _SAVED["cli"] = cli.decompose
    _SAVED["modules"] = (rs, tenring, est, cli)
    for n, fn in names.items():
        setattr(rs, n, fn)
        if n in _SAVED["package"]:
            setattr(tenring, n, fn)
    rs._SOLVERS.update(wrapped)
    est.decompose = decompose
    cli.decompose = decompose


def uninstall():
    """Restore the reference's own solvers."""
    if not _SAVED:
        return
    rs, tenring, est, cli = _SAVED["modules"]
    saved = _SAVED["solvers"]
    rs._SOLVERS.clear()
    rs._SOLVERS.update(saved.pop("_SOLVERS"))
    for n, fn in saved.items():
        setattr(rs, n, fn)
    for n, fn in _SAVED["package"].items():
        setattr(tenring, n, fn)
    est.decompose = _SAVED["estimator"]
    cli.decompose = _SAVED["cli"]
    _SAVED.clear()
