"""Time the fp64 environment product alone at a BASELINE shape (default c5 phase L:
25600 x 25600 x 400) on both engines, with nvidia-smi clocks/power sampled while it runs.
    python tools/oz_probe64.py [pre post r reps]"""
import json
import subprocess
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2210_11362_b200 import _lib as L  # noqa: E402

pre, post, r, reps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (25600, 25600, 20, 20)))
lib = L.lib()
torch.manual_seed(0)
x = torch.randn(pre, post, dtype=torch.float64, device="cuda")
H = torch.randn(post, r * r, dtype=torch.float64, device="cuda")
out = torch.empty(pre * r * r, dtype=torch.float64, device="cuda")
s = int(torch.cuda.current_stream().cuda_stream)
dig = torch.empty(lib.trals_oz64_digits_bytes(pre, post), dtype=torch.int8, device="cuda")
ex = torch.empty(pre, dtype=torch.int32, device="cuda")
sws = torch.empty(pre, dtype=torch.float64, device="cuda")
L.check(lib.trals_oz64_split_f64(x.data_ptr(), pre, post, 0, dig.data_ptr(), ex.data_ptr(), sws.data_ptr(), pre, s), "split")
wso = torch.empty(lib.trals_env_oz64_ws_elems(pre, post, 0, r, r), dtype=torch.float64, device="cuda")
wsd = torch.empty(max(lib.trals_gemm_ws_elems(1, pre, post, r * r), 1), dtype=torch.float64, device="cuda")


def oz():
    L.check(lib.trals_env_oz64(dig.data_ptr(), ex.data_ptr(), pre, post, 0, H.data_ptr(), r, r, out.data_ptr(), 0,
                               wso.data_ptr(), wso.numel(), s), "oz")


def dmma():
    L.check(lib.trals_env_f64(x.data_ptr(), pre, post, 0, H.data_ptr(), r, r, out.data_ptr(), 0, wsd.data_ptr(),
                              wsd.numel(), s), "dmma")


def sample(rows, stop):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append(line.strip())
    p.terminate()


for name, fn in (("ozaki", oz), ("dmma", dmma)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(rows, stop))
    th.start()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    e[0].record()
    for i in range(reps):
        fn()
        e[i + 1].record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = [e[i].elapsed_time(e[i + 1]) for i in range(reps)]
    clk = [float(v.split(",")[0]) for v in rows if v.split(",")[0].strip().replace(".", "").isdigit()]
    pw = [float(v.split(",")[1]) for v in rows if v.split(",")[1].strip().replace(".", "").isdigit()]
    print(json.dumps({"engine": name, "shape": [pre, post, r * r], "ms_min": min(ms), "ms_med": float(np.median(ms)),
                      "tflops_fp64_eq": 2.0 * pre * post * r * r / (min(ms) * 1e-3) / 1e12,
                      "sm_mhz_med": float(np.median(clk)) if clk else None,
                      "sm_mhz_min": min(clk) if clk else None, "power_w_max": max(pw) if pw else None,
                      "reasons": sorted(set(v.split(",")[2].strip() for v in rows))}), flush=True)
