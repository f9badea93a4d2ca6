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
from .ring import (Mode2Qr, gram_chain, gram_chain_order, lateral_gram, mode2_qr, random_cores, reconstruct,
                   subchain_merge, subchain_skip, tr_inner, tr_norm, validate_cores)
from .solvers import (BUCKETS, VARIANTS, AlsConfig, AlsReport, SweepCache, cheap_relative_error, decompose, tr_als,
                      tr_als_ne, tr_als_qr, tr_als_qrne)
from .synthetic import CORE_KINDS, SynthSpec, add_noise, make_dataset

__version__ = "0.1.0"

# the reference package's names (pkg/src/tenring/__init__.py:9-37) plus this package's extensions
__all__ = ["TensorRingALS", "Mode2Qr", "gram_chain", "gram_chain_order", "lateral_gram", "mode2_qr", "random_cores",
           "reconstruct", "subchain_merge", "subchain_skip", "tr_inner", "tr_norm", "validate_cores", "VARIANTS",
           "AlsConfig", "AlsReport", "cheap_relative_error", "decompose", "exact_relative_error", "tr_als",
           "tr_als_ne", "tr_als_qr", "tr_als_qrne", "SynthSpec", "add_noise", "make_dataset", "__version__",
           "SweepCache", "BUCKETS", "DegenerateTriangularError", "ElementBudgetError", "StaleCacheError", "CORE_KINDS",
           "read_tensor", "read_tensor_device", "write_tensor", "TensorFileError"]
