"""B200-native TR-ALS (NE / QR / QRNE) -- drop-in for the reference `tenring` solvers.

Public surface mirrors tenring's API for the path and its two sides
(pkg/src/tenring/__init__.py): AlsConfig, AlsReport, tr_als_ne, tr_als_qr,
tr_als_qrne, decompose; the TensorRingALS estimator; SynthSpec / make_dataset;
the .dten reader/writer (read_tensor_device lands X on the GPU).
The compute runs in libtrals.so (hand-written sm_100a kernels); importing this
package does not need a GPU, calling a solver does.
"""

from .errors import DegenerateTriangularError, ElementBudgetError, StaleCacheError
from .estimator import TensorRingALS, exact_relative_error
from .io import TensorFileError, read_tensor, read_tensor_device, write_tensor
from .solvers import (BUCKETS, VARIANTS, AlsConfig, AlsReport, decompose, tr_als, tr_als_ne, tr_als_qr,
                      tr_als_qrne)
from .synthetic import CORE_KINDS, SynthSpec, make_dataset

__version__ = "0.1.0"

__all__ = ["AlsConfig", "AlsReport", "decompose", "tr_als", "tr_als_ne", "tr_als_qr", "tr_als_qrne",
           "VARIANTS", "BUCKETS", "DegenerateTriangularError", "ElementBudgetError", "StaleCacheError",
           "TensorRingALS", "exact_relative_error", "SynthSpec", "make_dataset", "CORE_KINDS", "read_tensor",
           "read_tensor_device", "write_tensor", "TensorFileError", "__version__"]
