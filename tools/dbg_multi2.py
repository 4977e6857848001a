import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc
a = sp.laplacian_3d(12); h = sp.build_hierarchy(a, 6)
f = sp.factorize(a, h, 0.01, "second-full", skip_levels=2)
cl = orc.nd_hierarchy(a.n, a.row_ptr, a.col_idx, 6)
of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, 6, 0.01, "second-full", 2)
x = np.random.default_rng(0).standard_normal((a.n, 3))
r = of.apply_m(x)
z1 = np.column_stack([f.apply_m(x[:, j]) for j in range(3)])
print("1d vs oracle", np.linalg.norm(z1 - r) / np.linalg.norm(r))
for k in (1, 2, 3):
    z = f.apply_m(x[:, :k])
    print(k, "2d vs oracle", np.linalg.norm(z - r[:, :k]) / np.linalg.norm(r[:, :k]))
print(type(f.plan).__name__)
