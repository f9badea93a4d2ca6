"""Device time of the per-core Householder QR (trals_core_qr_f64) at the BASELINE core shapes, graph-replayed."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_11362_b200 import _lib as L  # noqa: E402
from tools.time_solve import graph_time  # noqa: E402

lib = L.lib()
for I, RR in [(100, 25), (64, 64), (500, 100), (40, 64), (160, 400), (30, 9), (2, 9)]:
    g = torch.from_numpy(np.random.default_rng(I + RR).standard_normal((I, RR))).cuda()
    k = min(I, RR)
    R = torch.empty((k, RR), dtype=torch.float64, device="cuda")
    ws = torch.empty(max(1, lib.trals_core_qr_ws_elems(I, RR)), dtype=torch.float64, device="cuda")

    def qr():
        L.check(lib.trals_core_qr_f64(g.data_ptr(), I, RR, R.data_ptr(), ws.data_ptr(), ws.numel(),
                                      int(torch.cuda.current_stream().cuda_stream)), "qr")
    t = graph_time(qr)
    r_ref = np.linalg.qr(g.cpu().numpy(), mode="r")
    r_ref = r_ref * np.where(np.diag(r_ref) < 0, -1.0, 1.0)[:, None]
    err = float(np.linalg.norm(R.cpu().numpy() - r_ref) / np.linalg.norm(r_ref))
    print(json.dumps({"I": I, "RR": RR, "qr_us": round(t, 1), "rel_err_vs_lapack": err}))
