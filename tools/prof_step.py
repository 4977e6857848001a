"""Where the wall time of one bench step goes (host view)."""
import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
a, b, lv = sp.baseline_problem("C4")
h = sp.build_hierarchy(a, lv)
bd = torch.from_numpy(b).cuda()
def step():
    f = sp.factorize(a, h, 1e-2, "second-full")
    x, rep = sp.pcg(a, bd, m=f.apply_m, tol=1e-12)
    return f, rep
for _ in range(2):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
f, rep = step()
torch.cuda.synchronize()
pr.disable()
print("step", time.perf_counter() - t0, f.timings, rep.solve_seconds)
pstats.Stats(pr).sort_stats("cumtime").print_stats(30)
