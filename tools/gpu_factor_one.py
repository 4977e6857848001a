import sys, time, traceback
import numpy as np
sys.path.insert(0, '.')
import paper_2007_00789_b200 as sp
from tests.golden_cases import load, matrix_for
tag = sys.argv[1]
rec, arr = load(tag)
a = matrix_for(tag)
h = sp.build_hierarchy(a, rec["levels"])
f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"])
got = [[[e["cluster"], e["size_before"], e["size_after"], e["rank_f2"]] for e in lv["interfaces"]] for lv in f.diagnostics["levels"]]
want = [lv["interfaces"] for lv in rec["diagnostics"]]
print("ranks ok", got == want)
