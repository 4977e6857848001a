"""RRQR wave times of two consecutive factorizations in one process
(first vs warm)."""
import json, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine as E
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
for it in range(3):
    E.WAVE_LOG = []
    f = sp.factorize(a, h, 1e-2, "second-full")
    torch.cuda.synchronize()
    ms = [e0.elapsed_time(e1) for (cnt, grid, vmax, e0, e1, sl) in E.WAVE_LOG]
    print(json.dumps({"iter": it, "rrqr_total_ms": round(sum(ms), 1), "first5": [round(x, 1) for x in ms[:5]],
                      "top3": sorted([round(x, 1) for x in ms])[-3:]}))
