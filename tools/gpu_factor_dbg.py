import sys, time, traceback
import numpy as np
sys.path.insert(0, '.')
import paper_2007_00789_b200 as sp
from tests.golden_cases import load, matrix_for, small_tags
for tag in small_tags():
    try:
        rec, arr = load(tag)
        a = matrix_for(tag)
        h = sp.build_hierarchy(a, rec["levels"])
        t0 = time.time()
        f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"])
        t1 = time.time()
        got = [[[e["cluster"], e["size_before"], e["size_after"], e["rank_f2"]] for e in lv["interfaces"]] for lv in f.diagnostics["levels"]]
        want = [lv["interfaces"] for lv in rec["diagnostics"]]
        x, rep = sp.pcg(a, arr["b"], m=f.apply_m, tol=rec["tol"])
        print(tag, "ranks_ok", got == want, "ncg", rep.n_cg, rec["n_cg"], "nnz", f.nnz_factor, rec["nnz_factor"], "t", round(t1-t0,3), f.timings, flush=True)
        if got != want:
            for g, w in zip(got, want):
                if g != w: print("  got", g[:6], "\n  want", w[:6]); break
    except Exception:
        traceback.print_exc()
