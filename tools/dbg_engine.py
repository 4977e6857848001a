import sys, numpy as np
sys.path.insert(0, '.')
import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc
a = sp.laplacian_2d(8)
h = sp.build_hierarchy(a, 3)
skip = int(sys.argv[1])
f = sp.factorize(a, h, 0.1, "first", skip_levels=skip)
cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, 3, 0.1, "first", skip)
print("nops", len(f.ops), len(of.ops))
for x, y in zip(f.ops, of.ops):
    errs = []
    for nm in ("lower", "panel", "q"):
        if hasattr(y, nm) and getattr(y, nm) is not None and hasattr(x, nm):
            gx, gy = getattr(x, nm), getattr(y, nm)
            errs.append((nm, gx.shape == gy.shape and float(np.abs(gx-gy).max()) if gx.size else 0))
    print(x.kind.value, errs, flush=True)
print(f.diagnostics["levels"])
