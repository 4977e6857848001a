import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine as E
a, b, lv = sp.baseline_problem("C4")
h = sp.build_hierarchy(a, 15)
f = sp.factorize(a, h, 1e-2, "second-full")
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter()
f = sp.factorize(a, h, 1e-2, "second-full")
torch.cuda.synchronize()
t1 = time.perf_counter()
p = f.plan
torch.cuda.synchronize()
t2 = time.perf_counter()
pr.disable()
print("factorize", t1 - t0, "plan", t2 - t1, f.timings)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
