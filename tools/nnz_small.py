"""nnz_factor of the device factor against every small golden (difference
and number of orthogonal operators)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.golden_cases import hierarchy_for, load, matrix_for, small_tags, config_tags
import paper_2007_00789_b200 as sp
tags = small_tags() + [t for t in config_tags() if "--all" in sys.argv]
for tag in tags:
    rec, _ = load(tag)
    a = matrix_for(tag)
    h = hierarchy_for(tag, a, rec["levels"])
    f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"], digest=False)
    nq = sum(1 for op in f.ops if op.kind.value == "orthogonal")
    d = f.nnz_factor - rec["nnz_factor"]
    print(f"{tag:50s} nnz {rec['nnz_factor']:12d} diff {d:8d} rel {d / rec['nnz_factor']:.2e} n_q {nq}", flush=True)
