import sys, numpy as np
sys.path.insert(0, '.')
from oracle import spand_oracle as orc
from paper_2007_00789_b200.rrqr import rrqr_single
rng = np.random.default_rng(0)
m, n, g = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, n)))
r = rrqr_single(a, 1e-2, "second-full", group=g)
ref = orc.sparsify_panel(a, 1e-2, "second-full")
print(m, n, g, "rank", r.rank_c, ref["rank_c"], flush=True)
