"""Per-step device time of one sweep (each engine step serialised and bracketed by
CUDA events on its own stream), for finding what besides the environment GEMMs
costs time on the small configs.

    python tools/step_profile.py c4 [ne|qr|qrne] [float64|float32]
"""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    variant = sys.argv[2] if len(sys.argv) > 2 else "ne"
    dtype = sys.argv[3] if len(sys.argv) > 3 else "float64"
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
    x, _ = make_dataset_device(order, dim, rt, noise, sd)
    if dtype == "float32":
        x = x.float()
    eng = SweepEngine(x, [dim] * order, [rf] * order, variant)
    eng.prepare_x()
    eng.compute_xnorm2()
    eng.set_cores(random_cores([dim] * order, [rf] * order, make_rng(si)))
    for _ in range(3):
        eng.run_sweep()
    torch.cuda.synchronize()
    times = []
    for st in eng.steps:
        if st.kind in ("fork", "join"):
            continue
        eng._cur = eng.side if st.stream == "side" else None
        s = eng.side if st.stream == "side" else eng.stream
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        st.fn()
        b.record(s)
        torch.cuda.synchronize()
        times.append((st.bucket, st.name, st.stream, a.elapsed_time(b) * 1e3))
    eng._cur = None
    total = sum(t for *_, t in times)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for bucket, nm, stream, t in times:
        key = (bucket, nm.split("[")[0].split(" ")[0], stream)
        agg[key][0] += 1
        agg[key][1] += t
    print(f"{name} {variant} {dtype}: {len(times)} steps, serialised sum {total:.1f} us")
    for (bucket, nm, stream), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {bucket:9s} {nm:22s} {stream:5s} n={n:3d} {t:9.1f} us  ({t / total:5.1%})")
    print("  top single steps:")
    for bucket, nm, stream, t in sorted(times, key=lambda r: -r[3])[:12]:
        print(f"    {t:8.1f} us  {bucket:9s} {stream:5s} {nm}")


if __name__ == "__main__":
    main()
