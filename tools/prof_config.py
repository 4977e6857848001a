"""Per-kernel-class device time of one factorize + solve (CUDA events)."""
import json, sys, time
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import _lib
name, scheme, eps = sys.argv[1], sys.argv[2], float(sys.argv[3])
levels = int(sys.argv[4]) if len(sys.argv) > 4 else None
a, b, lv = sp.baseline_problem(name)
lv = levels or lv
h = sp.build_hierarchy(a, lv)
f = sp.factorize(a, h, eps, scheme)   # warm
with _lib.profile() as pf:
    t0 = time.perf_counter(); f = sp.factorize(a, h, eps, scheme); torch.cuda.synchronize(); tf = time.perf_counter() - t0
print(json.dumps({"factorize_s": tf, "timings": f.timings, "kernels": pf.result}))
x, r = sp.pcg(a, b, m=f.apply_m, tol=1e-12)
with _lib.profile() as pf:
    t0 = time.perf_counter(); x, r = sp.pcg(a, b, m=f.apply_m, tol=1e-12); ts = time.perf_counter() - t0
print(json.dumps({"solve_s": ts, "n_cg": r.n_cg, "kernels": pf.result}))
t0 = time.perf_counter(); plan = f.plan; print("plan_cached", time.perf_counter() - t0, "launches/apply", plan.launches)
