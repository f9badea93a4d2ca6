"""Exception types with the reference's class hierarchy (so callers' except-clauses keep working)."""

import numpy as np


class ElementBudgetError(MemoryError):
    """Dense tensor larger than the element budget (reference validation.py:12-14)."""


class DegenerateTriangularError(np.linalg.LinAlgError):
    """Triangular diagonal below the 1e-13 floor (reference linalg.py:23-33)."""

    def __init__(self, index, value, floor):
        self.index = int(index)
        self.value = float(value)
        self.floor = float(floor)
        super().__init__(
            f"triangular factor diagonal {value:.3e} at index {index} is below "
            f"the degeneracy floor {floor:.3e}")


class StaleCacheError(RuntimeError):
    """Cheap error requested from a non-fresh sweep cache (reference solvers.py:136-137)."""
