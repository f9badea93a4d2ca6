"""ncu fodder: one per-core Householder QR (trals_core_qr_f64) at I x RR (default 64 x 64)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import _lib as L  # noqa: E402

I, RR = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (64, 64)
lib = L.lib()
g = torch.from_numpy(np.random.default_rng(I + RR).standard_normal((I, RR))).cuda()
R = torch.empty((min(I, RR), RR), dtype=torch.float64, device="cuda")
ws = torch.empty(max(1, lib.trals_core_qr_ws_elems(I, RR)), dtype=torch.float64, device="cuda")
for _ in range(2):
    L.check(lib.trals_core_qr_f64(g.data_ptr(), I, RR, R.data_ptr(), ws.data_ptr(), ws.numel(), 0), "qr")
torch.cuda.synchronize()
print("ok")
