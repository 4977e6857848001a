import sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc
from tests.golden_cases import load, matrix_for
tag = sys.argv[1]
rec, arr = load(tag)
a = matrix_for(tag)
h = sp.build_hierarchy(a, rec["levels"])
f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"])
cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, rec["levels"], rec["eps"], rec["scheme"], rec["skip_levels"])
for i, (x, y, w) in enumerate(zip(f.ops, of.ops, rec["ops"])):
    if x.nnz != w["nnz"]:
        print(i, x.kind.value, x.nnz, w["nnz"], y.nnz)
        for nm in ("lower", "panel", "q", "e_tilde"):
            if hasattr(x, nm) and getattr(y, nm, None) is not None:
                gx, gy = getattr(x, nm), getattr(y, nm)
                dz = np.argwhere((gx != 0) != (gy != 0))
                print("  ", nm, gx.shape, "pattern diffs", len(dz), [(tuple(d), gx[tuple(d)], gy[tuple(d)]) for d in dz[:4]])
