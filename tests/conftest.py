import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return dict(np.load(path, allow_pickle=False))


def golden_cores(rec, prefix, n):
    return [rec[f"{prefix}_{j}"] for j in range(n)]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0))


@pytest.fixture(autouse=True, scope="module")
def _release_plans():
    """Drop the cached engines after every test module: the BASELINE-size plans keep tens of GB of
    device buffers (operand planes, workspaces) alive otherwise."""
    yield
    try:
        import gc

        import torch
        if torch.cuda.is_available():
            from paper_2210_11362_b200.solvers import clear_plan_cache
            clear_plan_cache()
            gc.collect()
            torch.cuda.empty_cache()
    except Exception:
        pass
