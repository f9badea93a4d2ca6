"""Run the exact-error residual (fused reconstruct + (X - X_hat)^2, trals_residual_oz64) of one c5 sweep
inside cudaProfilerStart/Stop (for `ncu --profile-from-start off`), or time it with CUDA events."""
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
mode = sys.argv[2] if len(sys.argv) > 2 else "profile"
order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
x, _ = make_dataset_device(order, dim, rt, noise, sd)
eng = SweepEngine(x, x.shape, [rf] * order, "ne", fp64_gemm="ozaki")
eng.prepare_x()
eng.compute_xnorm2()
eng.set_cores(random_cores(x.shape, [rf] * order, make_rng(si)))
eng.run_sweep()
out = torch.zeros(3, dtype=torch.float64, device="cuda")
eng.error_step(out, exact=True)
torch.cuda.synchronize()
if mode == "profile":
    torch.cuda.profiler.start()
    eng.error_step(out, exact=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        eng.error_step(out, exact=True)
    b.record()
    torch.cuda.synchronize()
    print(f"exact error step: {a.elapsed_time(b) / 10:.3f} ms, e = {out[0].item()!r}")
print("ok")
