"""Time the X-streaming environment steps of one sweep (CUDA events, median of reps)."""
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
x, _ = make_dataset_device(order, dim, rt, noise, sd)
eng = SweepEngine(x, x.shape, [rf] * order, "ne", fp64_gemm="ozaki")
eng.prepare_x()
eng.compute_xnorm2()
eng.set_cores(random_cores(x.shape, [rf] * order, make_rng(si)))
eng.run_sweep()
torch.cuda.synchronize()
out = []
for st in eng.steps:
    if st.kind != "op":
        continue
    eng._cur = eng.side if st.stream == "side" else None
    if st.name.startswith("env"):
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            st.fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        out.append(f"{st.name} {ts[len(ts) // 2] * 1000:.1f}us")
    else:
        st.fn()
    eng._cur = None
torch.cuda.synchronize()
print(name, " ".join(out))
