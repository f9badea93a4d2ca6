"""Device time of the small dense kernels (Cholesky, solve) at the BASELINE sizes, replayed from a CUDA graph
(so host/ctypes overhead between launches is excluded)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import ops  # noqa: E402


def graph_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        fn()
        g.capture_end()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def _main():
    import os
    sizes = [(int(v), 64) for v in os.environ['SIZES'].split(',')] if os.environ.get('SIZES') else [(25, 100), (64, 64), (100, 500), (64, 40), (400, 160)]
    for m, rows in sizes:
        rng = np.random.default_rng(m)
        a = rng.standard_normal((2 * m, m))
        s = torch.from_numpy(a.T @ a).cuda()
        M = torch.from_numpy(rng.standard_normal((rows, m))).cuda()
        f = ops.cholesky(s)
        Z = ops.chol_solve(f, M)
        from paper_2210_11362_b200 import _lib as L
        lib = L.lib()
        wsz = ops.ws(lib.trals_chol_solve_ws_elems(rows, m), s.device)

        def chol():
            L.check(lib.trals_cholesky_f64(s.data_ptr(), m, f.U.data_ptr(), f.L.data_ptr(), f.aux.data_ptr(), 0,
                                           f.info.data_ptr(), int(torch.cuda.current_stream().cuda_stream)), "chol")

        def solve():
            L.check(lib.trals_chol_solve_f64(f.U.data_ptr(), f.L.data_ptr(), f.aux.data_ptr(), m, M.data_ptr(), rows,
                                             Z.data_ptr(), wsz.data_ptr(), wsz.numel(),
                                             int(torch.cuda.current_stream().cuda_stream)), "solve")
        print(json.dumps({"m": m, "rows": rows, "cholesky_us": round(graph_time(chol), 1),
                          "chol_solve_us": round(graph_time(solve), 1)}))


if __name__ == '__main__':
    _main()
