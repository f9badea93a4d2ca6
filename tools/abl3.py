"""Is the (non-firing) fallback launch slow by itself or by its position? Replace it by a tiny relayout."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.ablate as A  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200 import _lib as L  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402

order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
x, _ = make_dataset_device(order, dim, rt, noise, sd)
eng = SweepEngine(x, [dim] * order, [rf] * order, "ne")
eng.compute_xnorm2()
eng.set_cores(random_cores([dim] * order, [rf] * order, make_rng(si)))
lib = eng.lib
a = torch.zeros(64, dtype=torch.float64, device="cuda")
b = torch.zeros(64, dtype=torch.float64, device="cuda")


class Swap:
    def __init__(self, real, mode):
        self.real, self.mode = real, mode

    def __getattr__(self, k):
        f = getattr(self.real, k)
        if k == "trals_spd_fallback_f64":
            def g(*args):
                sp = args[-1]
                if self.mode == "relayout":
                    return self.real.trals_core_relayout_f64(a.data_ptr(), 0, 2, 4, 2, b.data_ptr(), 1, sp)
                if self.mode == "skip":
                    return 0
                return f(*args)
            return g
        return f


out = {}
for mode in ("real", "relayout", "skip"):
    eng.lib = Swap(lib, mode)
    out[mode] = A.timed(eng, [])
eng.lib = lib
print(json.dumps(out))
