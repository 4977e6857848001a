import sys, numpy as np
sys.path.insert(0, '.')
from oracle import spand_oracle as orc
from paper_2007_00789_b200 import rrqr_sparsify
from paper_2007_00789_b200.rrqr import rrqr_single
mode = sys.argv[1]
rng = np.random.default_rng(0)
for (m, n, g) in [(5, 8, 1), (12, 20, 1), (12, 20, 2), (30, 100, 3), (64, 300, 4)]:
    a = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, n)))
    if mode == "single":
        r = rrqr_single(a, 1e-2, "second-full", group=g)
    ref = orc.sparsify_panel(a, 1e-2, "second-full")
    print(m, n, g, "rank", r.rank_c, ref["rank_c"], "qc", np.abs(np.abs(r.q_c) - np.abs(ref["q_c"])).max() if r.rank_c == ref["rank_c"] else None,
          "rc", np.abs(r.r_coarse - ref["r_coarse"]).max() if r.rank_c == ref["rank_c"] else None, flush=True)
