"""Per-launch timing of the grouped GEMM inside one C4-L15 factorization."""
import json, sys
sys.path.insert(0, '.')
import torch
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import _lib
name, levels = sys.argv[1], int(sys.argv[2])
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
sp.factorize(a, h, 1e-2, "second-full")
rec = []
orig = _lib.call
def call(nm, *args):
    if nm == "spand_gemm_grouped":
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); r = orig(nm, *args); e1.record()
        rec.append((args[0], args[8], args[9], e0, e1))
        return r
    return orig(nm, *args)
_lib.call = call
import paper_2007_00789_b200.engine as E
E._lib.call = call
f = sp.factorize(a, h, 1e-2, "second-full")
torch.cuda.synchronize()
rows = [(nt, bT, lo, e0.elapsed_time(e1)) for nt, bT, lo, e0, e1 in rec]
tot = sum(r[3] for r in rows)
print(json.dumps({"gemm_ms": tot, "launches": len(rows)}))
import collections
buck = collections.defaultdict(lambda: [0, 0.0, 0])
for nt, bT, lo, ms in rows:
    k = 1 << max(0, (nt - 1).bit_length())
    buck[k][0] += 1; buck[k][1] += ms; buck[k][2] += nt
for k in sorted(buck):
    print(f"tiles<= {k:8d}: launches {buck[k][0]:5d} ms {buck[k][1]:8.2f} tiles {buck[k][2]}")
for r in sorted(rows, key=lambda r: -r[3])[:15]:
    print(r)
