"""Time the int8 environment GEMM (trals_env_oz) alone on the c4 shapes (probe)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_11362_b200 import _lib as L  # noqa: E402


def main():
    lib = L.lib()
    for pre, post, side in [(64000, 1600, 0), (1600, 64000, 1), (1600, 64000, 0), (64000, 1600, 1)]:
        r_lo = r_hi = 8
        x = torch.randn(pre, post, dtype=torch.float32, device="cuda")
        rows, K = (pre, post) if side == 0 else (post, pre)
        H = torch.randn(K, r_lo * r_hi, dtype=torch.float64, device="cuda")
        d = torch.empty(lib.trals_oz_digits_bytes(rows, K), dtype=torch.int8, device="cuda")
        e = torch.empty(rows, dtype=torch.int32, device="cuda")
        sws = torch.empty(lib.trals_oz_split_ws_elems(pre, post, side), dtype=torch.float64, device="cuda")
        s = int(torch.cuda.current_stream().cuda_stream)
        L.check(lib.trals_oz_split_f32(x.data_ptr(), pre, post, side, d.data_ptr(), e.data_ptr(), sws.data_ptr(),
                                       sws.numel(), s), "split")
        E = torch.empty(rows * r_lo * r_hi, dtype=torch.float64, device="cuda")
        ws = torch.empty(lib.trals_env_oz_ws_elems(pre, post, side, r_lo, r_hi), dtype=torch.float64, device="cuda")

        def run():
            L.check(lib.trals_env_oz(d.data_ptr(), e.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi,
                                     E.data_ptr(), 0, ws.data_ptr(), ws.numel(), s), "env")
        for _ in range(3):
            run()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 20
        print(f"pre={pre} post={post} side={side}: {ms * 1e3:.1f} us "
              f"({pre * post * 4 / ms / 1e6:.0f} GB/s of digits)", flush=True)
        del x, d


if __name__ == "__main__":
    main()
