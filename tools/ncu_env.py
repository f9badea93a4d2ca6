"""Run the two X-streaming environment GEMMs of a sweep inside cudaProfilerStart/Stop
(for `ncu --profile-from-start off`), everything else outside the capture window."""
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
fp64_gemm = sys.argv[2] if len(sys.argv) > 2 else "ozaki"
order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
x, _ = make_dataset_device(order, dim, rt, noise, sd)
eng = SweepEngine(x, x.shape, [rf] * order, "ne", fp64_gemm=fp64_gemm)
eng.prepare_x()
eng.compute_xnorm2()
eng.set_cores(random_cores(x.shape, [rf] * order, make_rng(si)))
eng.run_sweep()
torch.cuda.synchronize()
for st in eng.steps:
    if st.kind != "op":
        continue
    if st.name.startswith("env"):
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        st.fn()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    else:
        eng._cur = eng.side if st.stream == "side" else None
        st.fn()
        eng._cur = None
torch.cuda.synchronize()
print("ok")
