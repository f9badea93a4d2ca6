"""B200-native TR-ALS (NE / QR / QRNE) -- drop-in for the reference `tenring` solvers.

Public surface mirrors tenring's solver API (pkg/src/tenring/__init__.py):
AlsConfig, AlsReport, tr_als_ne, tr_als_qr, tr_als_qrne, decompose.
The compute runs in libtrals.so (hand-written sm_100a kernels); importing this
package does not need a GPU, calling a solver does.
"""

from .errors import DegenerateTriangularError, ElementBudgetError, StaleCacheError
from .solvers import (BUCKETS, VARIANTS, AlsConfig, AlsReport, decompose, tr_als, tr_als_ne, tr_als_qr,
                      tr_als_qrne)

__version__ = "0.1.0"

__all__ = ["AlsConfig", "AlsReport", "decompose", "tr_als", "tr_als_ne", "tr_als_qr", "tr_als_qrne",
           "VARIANTS", "BUCKETS", "DegenerateTriangularError", "ElementBudgetError", "StaleCacheError",
           "__version__"]
