import sys, torch
sys.path.insert(0, ".")
from bench import CONFIGS
from paper_2210_11362_b200.engine import SweepEngine
from paper_2210_11362_b200.host import make_rng, random_cores
from paper_2210_11362_b200.synthetic import make_dataset_device
order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS["c5"]
x, _ = make_dataset_device(order, dim, rt, noise, sd)
eng = SweepEngine(x, [dim]*order, [rf]*order, "ne")
eng.prepare_x(); eng.compute_xnorm2(); eng.set_cores(random_cores([dim]*order, [rf]*order, make_rng(si)))
out = torch.zeros(3, dtype=torch.float64, device="cuda")
for exact in (False, True):
    eng.run_sweep(); eng.error_step(out, exact=exact); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True); c = torch.cuda.Event(enable_timing=True)
    a.record(); eng.run_sweep(); b.record(); eng.error_step(out, exact=exact); c.record(); torch.cuda.synchronize()
    print("exact" if exact else "cheap", "sweep ms", a.elapsed_time(b), "error ms", b.elapsed_time(c), "err", float(out[0]))
