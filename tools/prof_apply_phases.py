"""Per-phase timing of the structured apply (eager launches, CUDA events)."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import _lib
from paper_2007_00789_b200.device import ptr, stream
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
torch.cuda.synchronize()
t0 = time.perf_counter(); plan = f.plan; torch.cuda.synchronize(); t_plan = time.perf_counter() - t0
print("plan_s", t_plan, getattr(plan, "build_times", None), "image MB", plan.image_host.nbytes / 1e6)
img = plan.image_host
ph = plan.phase_table
x = torch.from_numpy(b).cuda()
plan.run(x.clone()); torch.cuda.synchronize()
rows = []
st = stream()
for rep in range(3):
    xb = plan.xbuf
    evs = []
    for k, (tasks, tiles, ntile, chunks, nch, contrib, grid) in enumerate(plan.fwd + plan.bwd):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        _lib.call("spand_gemv_items", ntile, grid, tiles, tasks, ptr(xb), plan.n, ptr(plan.scratch), plan.scratch_len, 1, st)
        e1.record()
        _lib.call("spand_apply_runs", nch, chunks, contrib, ptr(xb), plan.n, ptr(plan.scratch), plan.scratch_len, 1, st)
        e2.record()
        evs.append((e0, e1, e2))
    torch.cuda.synchronize()
    times = [(a0.elapsed_time(a1), a1.elapsed_time(a2)) for a0, a1, a2 in evs]
nf = len(plan.fwd)
tot_g = tot_s = 0.0
out = []
for k, (tg, ts) in enumerate(times):
    to, nt, tio, ntile, co, nch, cbo, _, _, used = ph[k].tolist()
    tr = img[to:to + 8 * nt].reshape(-1, 8)
    mb = float((tr[:, 2] * tr[:, 3]).sum()) * 8
    tot_g += tg; tot_s += ts
    out.append({"k": k, "dir": "f" if k < nf else "b", "ntask": nt, "ntile": ntile, "nchunk": nch,
                "mat_MB": mb / 1e6, "gemv_us": tg * 1000, "runs_us": ts * 1000,
                "gemv_GBs": mb / (tg / 1000) / 1e9 if tg > 0 else None})
print(json.dumps({"phases": len(times), "gemv_ms": tot_g, "runs_ms": tot_s}))
out.sort(key=lambda r: -(r["gemv_us"] + r["runs_us"]))
for r in out[:40]:
    print(json.dumps(r))
# histogram by ntile
small = [r for r in out if r["ntile"] < 148]
print("phases with <148 tiles:", len(small), "time ms", sum(r["gemv_us"] + r["runs_us"] for r in small) / 1000)
x2 = x.clone(); f.apply_m_device(x2); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f.apply_m_device(x2)
e1.record(); torch.cuda.synchronize()
print("graph apply ms", e0.elapsed_time(e1) / 10)
