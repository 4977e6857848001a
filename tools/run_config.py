"""Run one BASELINE config on the GPU and compare with its golden (if any)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
name, scheme, eps = sys.argv[1], sys.argv[2], float(sys.argv[3])
levels = int(sys.argv[4]) if len(sys.argv) > 4 else None
a, b, lv = sp.baseline_problem(name)
lv = levels or lv
t0 = time.perf_counter(); h = sp.build_hierarchy(a, lv); t_h = time.perf_counter() - t0
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = sp.factorize(a, h, eps, scheme)
    torch.cuda.synchronize(); t_f = time.perf_counter() - t0
    x, r = sp.pcg(a, b, m=f.apply_m, tol=1e-12)
    print(json.dumps({"rep": rep, "t_hier": t_h, "t_factor": t_f, "timings": f.timings, "n_cg": r.n_cg, "t_solve": r.solve_seconds, "nnz": f.nnz_factor, "mu": f.nnz_factor / a.nnz, "true_res": r.true_residual}), flush=True)
tag = f"{name}_L{lv}_e{eps:g}_{scheme}"
p = os.path.join("tests/golden", tag + ".json")
if os.path.exists(p):
    rec = json.load(open(p))
    got = [[[e["cluster"], e["size_before"], e["size_after"], e["rank_f2"]] for e in l["interfaces"]] for l in f.diagnostics["levels"]]
    want = [l["interfaces"] for l in rec["diagnostics"]]
    nd = sum(1 for g, w in zip(got, want) for x, y in zip(g, w) if x != y)
    print("golden", tag, "ranks_equal", got == want, "n_mismatch", nd, "n_cg_ref", rec["n_cg"], "nnz_ref", rec["nnz_factor"], "t_factor_ref", rec["t_factor_s"])
    if got != want:
        for l, (g, w) in enumerate(zip(got, want)):
            for x, y in zip(g, w):
                if x != y:
                    print("  level", l, "got", x, "want", y)
