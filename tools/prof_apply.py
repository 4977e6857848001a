import json, sys, time
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import _lib
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
t0 = time.perf_counter(); plan = f.plan; t_plan = time.perf_counter() - t0
bd = torch.from_numpy(b).cuda()
x = bd.clone(); f.apply_m_device(x); torch.cuda.synchronize()
z_eager = bd.clone(); plan.run(z_eager); torch.cuda.synchronize()
print("graph vs eager", float((x - z_eager).abs().max()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f.apply_m_device(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
from paper_2007_00789_b200.metrics import apply_bytes
B = apply_bytes(f.nnz_factor, a.n)
print(json.dumps({"plan_s": t_plan, "launches": plan.launches, "apply_ms_graph": ms, "GBs": B / ms / 1e6, "B_apply_GB": B / 1e9}))
t0 = time.perf_counter(); xs, rep = sp.pcg(a, bd, m=f.apply_m, tol=1e-12); torch.cuda.synchronize()
print("pcg", rep.n_cg, time.perf_counter() - t0)
