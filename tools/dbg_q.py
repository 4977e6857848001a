import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc
from tests.golden_cases import load, matrix_for
tag = "lap3d_d8_L6_e0.01_k1_second-superfine"
rec, arr = load(tag)
a = matrix_for(tag)
h = sp.build_hierarchy(a, rec["levels"])
f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"])
cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, rec["levels"], rec["eps"], rec["scheme"], rec["skip_levels"])
for i, (x, y) in enumerate(zip(f.ops, of.ops)):
    if x.kind.value == "orthogonal":
        q = x.q
        m = q.shape[0]
        kc = y.k_c
        piv = y.pivots
        d = np.abs(np.abs(q) - np.abs(y.q)).max()
        if d > 1e-6:
            print("op", i, "m", m, "kc", kc, "len piv", len(piv), "maxdiff", d)
            # which columns differ
            cols = [j for j in range(m) if np.abs(np.abs(q[:, j]) - np.abs(y.q[:, j])).max() > 1e-6]
            print(" differing cols", cols[:20], "n", len(cols))
            print(" pivots", np.round(piv[:12], 6))
            break
# summary: count differing orthogonal ops
nd = 0
for i, (x, y) in enumerate(zip(f.ops, of.ops)):
    if x.kind.value == "orthogonal":
        if np.abs(np.abs(x.q) - np.abs(y.q)).max() > 1e-6:
            nd += 1
print("differing Q ops", nd)
