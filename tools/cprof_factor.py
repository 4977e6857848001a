import cProfile, pstats, sys, io
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
pr = cProfile.Profile(); pr.enable()
f = sp.factorize(a, h, 1e-2, "second-full"); torch.cuda.synchronize()
p = f.plan
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35); print(s.getvalue())
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue())
