"""Scikit-learn style estimator over the B200 solvers -- the reference's
`TensorRingALS` (pkg/src/tenring/estimator.py:16-130) with the same
parameters, attributes and methods, so `TensorRingALS(...).fit(X)` switches to
the GPU path unchanged (front-end wiring).

`fit` runs `decompose` on the device; `reconstruct` materialises the fitted
ring on the device (half chains + one DMMA GEMM) and returns a host array like
the reference; `score` is the negative exact relative error computed by the
fused residual kernel (X streamed once, X-hat never stored).
"""

from __future__ import annotations

import numbers

import numpy as np

from .host import check_dense_tensor, check_element_budget, check_ranks
from .solvers import VARIANTS, AlsConfig, decompose

try:  # the reference estimator derives from sklearn's BaseEstimator (get_params / set_params / clone)
    from sklearn.base import BaseEstimator
    from sklearn.exceptions import NotFittedError
except ImportError:  # pragma: no cover - sklearn is in this image; keep the class usable without it
    BaseEstimator = object

    class NotFittedError(ValueError, AttributeError):
        pass

__all__ = ["TensorRingALS", "exact_relative_error"]


def exact_relative_error(x, cores, budget=None):
    """||X - TR(cores)|| / ||X|| on the GPU (solvers.py:164-174 semantics): the
    reconstruction is fused into the residual reduction, never stored."""
    import torch

    from . import _lib as L
    from .engine import SweepEngine

    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dims = tuple(int(d) for d in t.shape)
    check_element_budget(dims, budget)
    cores = [np.asarray(g, dtype=np.float64) for g in cores]
    ranks = [int(g.shape[0]) for g in cores]
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_11362_b200 needs a CUDA device (no CPU fallback)")
    L.lib()
    xd = t.detach().to("cuda", torch.float64).contiguous()
    eng = SweepEngine(xd, dims, ranks, "ne", fp64_gemm="dmma")  # residual only: no digit planes
    xn = eng.compute_xnorm2()
    eng.set_cores(cores)
    out = torch.zeros(3, dtype=torch.float64, device=xd.device)
    eng.error_step(out, exact=True)
    if float(xn[0].item()) == 0.0:
        return 0.0
    return float(out[0].item())


class TensorRingALS(BaseEstimator):
    """Tensor-ring decomposition fitted by alternating least squares on a B200.

    Parameters and attributes are the reference's (estimator.py:16-72):
    rank, variant ('als' | 'ne' | 'qr' | 'qrne', all on the GPU), max_iter, tol, error_mode, random_state,
    rank_deficient_fallback, element_budget; fitted `cores_`, `errors_`,
    `n_iter_`, `report_`, `dims_`.  `dtype` (extension, default "float64")
    selects the fp32 variant.
    """

    def __init__(self, rank=5, variant="qrne", max_iter=20, tol=0.0, error_mode="exact", random_state=None,
                 rank_deficient_fallback=True, element_budget=None, dtype="float64"):
        self.rank = rank
        self.variant = variant
        self.max_iter = max_iter
        self.tol = tol
        self.error_mode = error_mode
        self.random_state = random_state
        self.rank_deficient_fallback = rank_deficient_fallback
        self.element_budget = element_budget
        self.dtype = dtype

    def _ranks_for(self, order):
        if isinstance(self.rank, numbers.Integral):
            return [int(self.rank)] * order
        return check_ranks(self.rank, order)

    def fit(self, X, y=None, init_cores=None):
        """Fit the decomposition to a dense tensor of order >= 2 (estimator.py:83-109)."""
        X = _as_checked(X)
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}; expected one of {VARIANTS}")
        config = AlsConfig(ranks=self._ranks_for(X.ndim), max_iters=self.max_iter, tol=self.tol,
                           seed=self.random_state, error_mode=self.error_mode,
                           rank_deficient_fallback=self.rank_deficient_fallback, init_cores=init_cores,
                           element_budget=self.element_budget, dtype=self.dtype)
        self.cores_, self.report_ = decompose(X, self.variant, config)
        self.errors_ = self.report_.errors
        self.n_iter_ = self.report_.n_iters
        self.dims_ = tuple(int(d) for d in X.shape)
        return self

    def _check_fitted(self):
        if not hasattr(self, "cores_"):
            raise NotFittedError("this TensorRingALS instance is not fitted yet; call fit first")

    def reconstruct(self):
        """Materialise the fitted low-rank tensor (estimator.py:117-120), built on the GPU."""
        self._check_fitted()
        from .synthetic import reconstruct_device
        check_element_budget([g.shape[1] for g in self.cores_], self.element_budget)
        return reconstruct_device(self.cores_).cpu().numpy()

    def score(self, X, y=None):
        """Negative relative reconstruction error, greater is better (estimator.py:122-130)."""
        self._check_fitted()
        X = _as_checked(X)
        if tuple(X.shape) != tuple(self.dims_):
            raise ValueError(f"X has shape {tuple(X.shape)}, fitted on {tuple(self.dims_)}")
        return -exact_relative_error(X, self.cores_, budget=self.element_budget)


def _as_checked(X):
    """check_dense_tensor(X, min_order=2) for host arrays; CUDA tensors are validated
    on the device by the solver (no host copy of a resident X)."""
    try:
        import torch
        if isinstance(X, torch.Tensor) and X.is_cuda:
            if X.dim() < 2:
                raise ValueError(f"tensor order {X.dim()} is below the minimum 2")
            if X.numel() == 0:
                raise ValueError("tensor has no elements")
            return X
    except ImportError:  # pragma: no cover
        pass
    return check_dense_tensor(X, min_order=2)
