"""Full-size parity on the BASELINE configurations (C2, C3, C4 at L11 and the
headline C4 at L15) against the reference's frozen outputs
(tests/golden/make_golden.py; the CPU reference takes up to 73 min per
config, so only size-independent properties are compared here):

- integer structure bit-exact: per-level interior counts, per-interface
  (cluster, size_before, size_after, rank_f2), the final block, the
  permutation (sha256) and the operator-kind string;
- nnz_factor within 2e-3 (exact-zero counting of rounding noise, see
  test_gpu_factorize.py);
- PCG: n_cg within +-1, same convergence flag, true residual within 10x of
  the reference's, and
  the first residual-history entries within 1e-6 relative of the
  reference's.
"""

import hashlib

import numpy as np
import pytest

from tests.golden_cases import config_tags, load, matrix_for, hierarchy_for

pytestmark = pytest.mark.gpu


def sha(arr):
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("tag", config_tags())
def test_config_matches_reference(tag):
    import paper_2007_00789_b200 as sp
    rec, arr = load(tag)
    a = matrix_for(tag)
    h = hierarchy_for(tag, a, rec["levels"])
    f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"])
    got = [[[e["cluster"], e["size_before"], e["size_after"], e["rank_f2"]]
            for e in lv["interfaces"]] for lv in f.diagnostics["levels"]]
    want = [lv["interfaces"] for lv in rec["diagnostics"]]
    assert got == want
    assert [lv["interior_clusters"] for lv in f.diagnostics["levels"]] == \
        [lv["interior_clusters"] for lv in rec["diagnostics"]]
    assert f.diagnostics["final_block"] == rec["final_block"]
    assert sha(np.asarray(f.perm, np.int64)) == rec["perm_sha"]
    kinds = "".join("GDQE"[["elimination", "scaling", "orthogonal",
                            "error-correction"].index(op.kind.value)] for op in f.ops)
    assert kinds == rec["op_kinds"]
    assert abs(f.nnz_factor - rec["nnz_factor"]) <= 2e-3 * rec["nnz_factor"] + 16
    b = arr["b"]
    x, rep = sp.pcg(a, b, m=f.apply_m, tol=rec["tol"])
    assert abs(rep.n_cg - rec["n_cg"]) <= 1
    assert rep.converged == rec["converged"]
    # the reference's true residual (high contrast: up to 16x the recursive one)
    assert rep.true_residual <= 10 * max(rec["true_residual"], rec["tol"])
    hist = np.asarray(rep.residual_history[:3])
    ref = np.asarray(rec["residual_history"][:3])
    assert np.allclose(hist, ref, rtol=1e-6, atol=0)
