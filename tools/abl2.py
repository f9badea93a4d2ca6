import os, sys, json, torch
sys.path.insert(0,'/root/repo')
import tools.ablate as A
from paper_2210_11362_b200 import _lib as L
from paper_2210_11362_b200.engine import SweepEngine
from paper_2210_11362_b200.host import make_rng, random_cores
from paper_2210_11362_b200.synthetic import make_dataset_device
from bench import CONFIGS
order, dim, rt, noise, sd, rf, si, sweeps = CONFIGS[sys.argv[1] if len(sys.argv)>1 else 'c2']
x,_=make_dataset_device(order, dim, rt, noise, sd)
eng=SweepEngine(x,[dim]*order,[rf]*order,'ne'); eng.compute_xnorm2(); eng.set_cores(random_cores([dim]*order,[rf]*order,make_rng(si)))
full=A.timed(eng, [])
lib=eng.lib
class Skip:
    def __init__(s, real, skip_layout): s.real=real; s.skip=skip_layout; s.n=0
    def __getattr__(s, k):
        f=getattr(s.real,k)
        if k=='trals_core_relayout_f64':
            def g(*a):
                if a[5]==s.skip and a[1]==L.LAYOUT_ZT: return 0
                return f(*a)
            return g
        return f
eng.lib=Skip(lib, L.LAYOUT_SLICE); t1=A.timed(eng, [])
eng.lib=Skip(lib, L.LAYOUT_C); t2=A.timed(eng, [])
eng.lib=lib
print(json.dumps({"full":full, "skip_ZT->SLICE":t1, "skip_ZT->C":t2}))
