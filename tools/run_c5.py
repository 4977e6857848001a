"""C5 (Q1 elasticity 24^3, node-blocked ND) on the GPU: factorize + PCG with
and without the six rigid-body modes preserved."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
a, b, lv, co = sp.c5_problem()
h = sp.build_hierarchy(a, lv, block=3)
r = sp.rigid_body_modes(co)
for nk in (None, r, None, r):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = sp.factorize(a, h, 0.01, "second-full", near_kernel=nk)
    torch.cuda.synchronize(); tf = time.perf_counter() - t0
    x, rep = sp.pcg(a, b, m=f.apply_m, tol=1e-12)
    kept = sum(e["size_after"] for lv_ in f.diagnostics["levels"] for e in lv_["interfaces"])
    print({"near_kernel": nk is not None, "factorize_s": round(tf, 3), "n_cg": rep.n_cg,
           "solve_s": round(rep.solve_seconds, 3), "true_res": rep.true_residual,
           "coarse_kept": kept, "nnz_factor": f.nnz_factor}, flush=True)
