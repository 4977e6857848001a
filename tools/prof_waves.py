"""Per-wave RRQR timing with panel statistics (m, n, k_stop)."""
import json, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine as E
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
try:
    sp.factorize(a, h, 1e-2, "second-full")  # warm
except Exception as exc:
    print("warm factorize raised", type(exc).__name__, exc)
E.WAVE_LOG = []
keep = {}
orig = E.Engine.collect
def col(self):
    keep["eng"] = self
    return orig(self)
E.Engine.collect = col
try:
    f = sp.factorize(a, h, 1e-2, "second-full")
except Exception as exc:
    print("factorize raised", type(exc).__name__, exc)
torch.cuda.synchronize()
eng = keep["eng"]
ev = eng.events.cpu().numpy().reshape(-1, E.EVENT_ROW)
# event row: p, m, n, k_stop, k_c, rank_f2, n_fine, ...
recs = []
tot = 0
for (cnt, grid, vmax, e0, e1, sl) in E.WAVE_LOG:
    ms = e0.elapsed_time(e1)
    tot += ms
    rows = ev[sl] if sl else np.zeros((0, E.EVENT_ROW), np.int64)
    m, n, ks = rows[:, 1], rows[:, 2], rows[:, 3]
    recs.append({"npanel": cnt, "grid": grid, "ms": round(ms, 3),
                 "m_max": int(m.max()) if len(m) else 0, "n_max": int(n.max()) if len(n) else 0,
                 "ks_max": int(ks.max()) if len(ks) else 0, "ks_sum": int(ks.sum()),
                 "frozen_frac": float(rows[:, 11].sum() / max(1, n.sum())),
                 "sum_mn_MB": float((m * n).sum()) * 8 / 1e6})
print(json.dumps({"rrqr_total_ms": tot, "launches": len(recs)}))
for r in sorted(recs, key=lambda r: -r["ms"])[:45]:
    print(json.dumps(r))
