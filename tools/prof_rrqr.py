import json, sys
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine
name, scheme, eps = sys.argv[1], sys.argv[2], float(sys.argv[3])
levels = int(sys.argv[4]) if len(sys.argv) > 4 else None
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels or lv)
sp.factorize(a, h, eps, scheme)
engine.WAVE_LOG = []
f = sp.factorize(a, h, eps, scheme)
torch.cuda.synchronize()
rows = []
for np_, grid, vmax, e0, e1 in engine.WAVE_LOG:
    ms = e0.elapsed_time(e1)
    rows.append((ms, np_, grid, vmax))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print("total_ms", tot, "waves", len(rows))
for r in rows[:25]:
    print(r)
# ranks of the big panels
for lv_ in f.diagnostics["levels"]:
    for e in lv_["margins"]:
        if e["size_before"] > 1000:
            print(lv_["level"], e["cluster"], e["size_before"], e["size_after"], e["k_stop"])
