"""Time one environment product (X . half chain) on each engine at a given shape, CUDA events.

    python tools/env_bench.py [--pre 25600 --post 25600 --r 20 --side 0 --reps 10] [--engines crt,oz64,dmma]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_11362_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pre", type=int, default=25600)
    ap.add_argument("--post", type=int, default=25600)
    ap.add_argument("--r", type=int, default=20)
    ap.add_argument("--side", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--engines", default="crt,oz64")
    a = ap.parse_args()
    lib = L.lib()
    pre, post, r, side = a.pre, a.post, a.r, a.side
    rows, K = (pre, post) if side == 0 else (post, pre)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    x = torch.randn((pre, post), dtype=torch.float64, device="cuda", generator=g)
    H = torch.randn((K, r * r), dtype=torch.float64, device="cuda", generator=g)
    s = int(torch.cuda.current_stream().cuda_stream)
    outs = {}
    for eng in a.engines.split(","):
        out = torch.empty(rows * r * r, dtype=torch.float64, device="cuda")
        if eng == "dmma":
            ws = torch.empty(max(lib.trals_gemm_ws_elems(1, rows, K, r * r), 1 << 22), dtype=torch.float64, device="cuda")

            def run():
                L.check(lib.trals_env_f64(x.data_ptr(), pre, post, side, H.data_ptr(), r, r, out.data_ptr(), 0,
                                          ws.data_ptr(), ws.numel(), s), "env")
            t_split = 0.0
        else:
            nbytes, split, split_ws, wsf, envf = {
                "crt": (lib.trals_crt_planes_bytes, lib.trals_crt_split_f64, lib.trals_crt_split_ws_elems,
                        lib.trals_env_crt_ws_elems, lib.trals_env_crt),
                "oz64": (lib.trals_oz64_digits_bytes, lib.trals_oz64_split_f64, lib.trals_oz_split_ws_elems,
                         lib.trals_env_oz64_ws_elems, lib.trals_env_oz64)}[eng]
            planes = torch.empty(nbytes(rows, K), dtype=torch.int8, device="cuda")
            exps = torch.empty(rows, dtype=torch.int32, device="cuda")
            sws = torch.empty(max(1, split_ws(pre, post, side)), dtype=torch.float64, device="cuda")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.check(split(x.data_ptr(), pre, post, side, planes.data_ptr(), exps.data_ptr(), sws.data_ptr(),
                          sws.numel(), s), "split")
            e1.record()
            torch.cuda.synchronize()
            t_split = e0.elapsed_time(e1)
            ws = torch.empty(wsf(pre, post, side, r, r), dtype=torch.float64, device="cuda")

            def run(planes=planes, exps=exps, ws=ws, envf=envf):
                L.check(envf(planes.data_ptr(), exps.data_ptr(), pre, post, side, H.data_ptr(), r, r, out.data_ptr(),
                             0, ws.data_ptr(), ws.numel(), s), "env")
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        outs[eng] = out
        rec = {"engine": eng, "pre": pre, "post": post, "r": r, "side": side, "env_ms": round(ms, 4),
               "split_ms": round(t_split, 3), "fp64_equiv_tflops": round(2.0 * rows * K * r * r / ms / 1e9, 2)}
        if eng != a.engines.split(",")[0]:
            first = outs[a.engines.split(",")[0]]
            rec["rel_vs_first"] = float((out - first).norm() / first.norm())
        print(json.dumps(rec), flush=True)
        if eng != "dmma":
            del planes, ws


if __name__ == "__main__":
    main()
