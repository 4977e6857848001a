import sys, time
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
torch.cuda.synchronize()
print("done", f.timings)
