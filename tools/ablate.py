"""Critical-path ablation of a sweep: graph-capture the sweep with some step kinds removed
and time the replay (timing only -- the numerics of an ablated sweep are meaningless).

    python tools/ablate.py c2 [ne]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2210_11362_b200.engine import SweepEngine  # noqa: E402
from paper_2210_11362_b200.host import make_rng, random_cores  # noqa: E402
from paper_2210_11362_b200.synthetic import make_dataset_device  # noqa: E402


def timed(eng, drop, reps=20):
    keep = eng.steps
    eng.steps = [st for st in keep if st.kind != "op" or not any(st.name.startswith(d) for d in drop)]
    try:
        g = eng.capture(with_error=False)
        for _ in range(3):
            eng.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        for _ in range(reps):
            eng.replay()
        b.record(eng.stream)
        torch.cuda.synchronize()
        del g
        return a.elapsed_time(b) / reps * 1e3
    finally:
        eng.steps = keep
        eng.graph = None


def main():
    if os.environ.get("PREFER_SHARED"):
        import ctypes
        import glob
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
            glob.glob("/usr/local/cuda/lib64/libcudart.so*")
        rt = ctypes.CDLL(cands[0])
        print("cudaDeviceSetCacheConfig ->", rt.cudaDeviceSetCacheConfig(2), cands[0])
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    variant = sys.argv[2] if len(sys.argv) > 2 else "ne"
    order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[name]
    x, _ = make_dataset_device(order, dim, rt, noise, sd)
    eng = SweepEngine(x, [dim] * order, [rf] * order, variant)
    eng.compute_xnorm2()
    eng.set_cores(random_cores([dim] * order, [rf] * order, make_rng(si)))
    names = sorted({st.name.rstrip("0123456789").split("[")[0].split(" ")[0] for st in eng.steps
                    if st.name and st.kind == "op"})
    out = {"config": name, "variant": variant, "full_us": timed(eng, [])}
    for nm in names:
        out[f"without_{nm}"] = timed(eng, [nm])
    out["without_env"] = timed(eng, ["env"])
    out["only_env"] = timed(eng, [n for n in names if n != "env"])
    print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
