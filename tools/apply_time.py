"""apply_m timing on one factor (CUDA graph replays, L2 flushed before):
ms per apply and B_apply GB/s; also the eager (non-graph) time."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
bd = torch.from_numpy(b).cuda()
x = bd.clone()
t0 = time.perf_counter(); f.apply_m_device(x); torch.cuda.synchronize()
first = time.perf_counter() - t0
flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
res = {}
for mode in ("eager", "graph"):
    if mode == "graph":
        for _ in range(40): f.apply_m_device(x)
    ts = []
    for _ in range(10):
        flush.zero_(); torch.cuda.synchronize()
        e0.record(); f.apply_m_device(x); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[mode] = round(float(np.median(ts)), 3)
B = 16.0 * f.nnz_factor + 32.0 * a.n
img = f.plan.build_times if hasattr(f.plan, "build_times") else {}
print(json.dumps({"apply_ms": res, "gbs_graph": B / (res["graph"] / 1e3) / 1e9, "B_apply_GB": B / 1e9,
                  "first_apply_s": first, "image": img,
                  "phases": int(len(f.plan.phase_table)) if hasattr(f.plan, "phase_table") else None}))
y = f.apply_m(b)
print("apply_m norm", float(np.linalg.norm(y)))
