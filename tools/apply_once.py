"""Factorize a BASELINE config and run ONE eager apply_m (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
plan = f.plan
x = torch.from_numpy(b).cuda()
torch.cuda.synchronize()
plan.run(x)
torch.cuda.synchronize()
print("done")
import json
img, ph = plan.image_host, plan.phase_table
stats = []
for r in ph.tolist():
    to, nt, io, ni, co, nch, cbo, grid, _, used = r
    tr = img[to:to + 8 * nt].reshape(-1, 8)
    stats.append({"ntask": nt, "nitem": ni, "grid": grid, "nchunk": nch,
                  "MB": float((tr[:, 2] * tr[:, 3]).sum()) * 8 / 1e6,
                  "trans_frac": float(tr[:, 4].mean()),
                  "max_rows": int(tr[:, 2].max()), "max_cols": int(tr[:, 3].max()),
                  "ncontrib": int(used)})
json.dump(stats, open("gpurun_out/phase_stats.json", "w"))
