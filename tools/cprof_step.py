"""cProfile of the host side of one warm resident step (factorize + PCG)."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
a, b, lv = sp.baseline_problem("C4")
h = sp.build_hierarchy(a, 15)
bd = torch.from_numpy(b).cuda()
def step():
    f = sp.factorize(a, h, 1e-2, "second-full")
    x, rep = sp.pcg(a, bd, m=f.apply_m, tol=1e-12)
    torch.cuda.synchronize()
step(); step()
cProfile.run("step()", "/tmp/step.prof")
st = pstats.Stats("/tmp/step.prof")
st.sort_stats("tottime").print_stats(25)
