import sys, time
sys.path.insert(0, '.')
import numpy as np, torch, ctypes
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import fastplan
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
torch.cuda.synchronize()
col = f._plan_factory.__closure__
t0 = time.perf_counter()
# replicate pieces
import paper_2007_00789_b200.engine as E
print({k: round(v, 3) for k, v in f.timings.items()})
orig = fastplan.NativeApplyPlan.__init__
ts = {}
lib = None
def wrap(fn, name):
    def g(*a, **k):
        t = time.perf_counter(); r = fn(*a, **k); torch.cuda.synchronize(); ts[name] = ts.get(name, 0) + time.perf_counter() - t; return r
    return g
fastplan.to_dev = wrap(fastplan.to_dev, "to_dev")
fastplan.to_dev_async = wrap(fastplan.to_dev_async, "to_dev_async")
t0 = time.perf_counter(); p = f.plan; torch.cuda.synchronize(); print("plan total", time.perf_counter() - t0, ts)
print(p.build_times)
