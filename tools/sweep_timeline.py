"""Timeline of one eager sweep as it really runs (main + side stream, joins included):
an event after every step on its own stream; prints each step's end time and the main
stream's increments, i.e. the critical path.

    python tools/sweep_timeline.py [c5] [ne] [auto|ozaki|dmma]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    variant = sys.argv[2] if len(sys.argv) > 2 else "ne"
    gemm = sys.argv[3] if len(sys.argv) > 3 else "auto"
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
    x, _ = make_dataset_device(order, dim, rt, noise, sd)
    eng = SweepEngine(x, [dim] * order, [rf] * order, variant, fp64_gemm=gemm)
    eng.prepare_x()
    eng.compute_xnorm2()
    eng.set_cores(random_cores([dim] * order, [rf] * order, make_rng(si)))
    err = torch.zeros(3, dtype=torch.float64, device="cuda")
    for _ in range(3):
        eng.run_sweep()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(eng.stream)
    marks = []
    for st in eng.steps:
        if st.kind == "fork":
            eng._fork_ev.record(eng.stream)
            eng.side.wait_event(eng._fork_ev)
            continue
        if st.kind == "join":
            eng._join_ev.record(eng.side)
            eng.stream.wait_event(eng._join_ev)
            continue
        eng._cur = eng.side if st.stream == "side" else None
        s = eng.side if st.stream == "side" else eng.stream
        st.fn()
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        marks.append((st.name, st.stream, e))
    eng._cur = None
    eng.error_step(err)
    e = torch.cuda.Event(enable_timing=True)
    e.record(eng.stream)
    marks.append(("error", "main", e))
    torch.cuda.synchronize()
    prev = 0.0
    print(f"{name} {variant} {eng.fp64_gemm}: step end times (us)")
    for nm, stream, ev in marks:
        t = t0.elapsed_time(ev) * 1e3
        if stream == "main":
            print(f"  {t:9.1f}  +{t - prev:8.1f}  main  {nm}")
            prev = t
        else:
            print(f"  {t:9.1f}             side  {nm}")


if __name__ == "__main__":
    main()
