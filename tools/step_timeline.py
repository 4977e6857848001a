"""Host/device timeline of one resident C4-L15 step (factorize + PCG), with
synchronisations at phase boundaries for attribution (so the total is a bit
above the bench's overlapped step)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine as E
a, b, lv = sp.baseline_problem("C4")
h = sp.build_hierarchy(a, 15)
bd = torch.from_numpy(b).cuda()
sch = sp.SchemeKind.from_string("second-full")
for rep in range(3):
    T = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng = E.Engine(a, h, 1e-2, sch, 4)
    T["symbolic"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    eng.run()            # ends with a synchronize
    T["run"] = time.perf_counter() - t1
    T.update({k: v for k, v in eng.timings.items() if k in ("launch_s", "plan_s")})
    TC = eng.timings
    t2 = time.perf_counter()
    ops, perm, diag, nnz = eng.collect()
    T["collect"] = time.perf_counter() - t2
    from paper_2007_00789_b200.factorize import Factorization
    f = Factorization(ops=ops, perm=perm, n=a.n, eps=1e-2, scheme=sch, skip_levels=4,
                      nnz_factor=int(nnz), diagnostics=diag, _keep=(eng.pool, eng.facbuf, eng.geo))
    f._plan = eng.apply_plan
    t3 = time.perf_counter()
    f._plan._ensure()
    torch.cuda.synchronize()
    T["apply_plan_wait"] = time.perf_counter() - t3
    t4 = time.perf_counter()
    x, rep_ = sp.pcg(a, bd, m=f.apply_m, tol=1e-12)
    torch.cuda.synchronize()
    T["pcg"] = time.perf_counter() - t4
    T["total"] = time.perf_counter() - t0
    print({k: round(v, 4) for k, v in T.items()}, "n_cg", rep_.n_cg, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in f._plan.build_times.items()},
          {k: round(v, 4) for k, v in TC.items() if k.startswith("collect")}, flush=True)
