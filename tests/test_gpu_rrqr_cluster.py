"""The clustered RRQR variant (rrqr.cu, ``spand_rrqr_wave_clustered``):
thread-block clusters that split each cluster's columns by rows over its
CTAs.  Same contract as the classic kernel: integer decisions (perm, k_c,
k_stop / rank_f2) identical to the CPU oracle (reference dense.py:117-222),
payloads within 1e-10 relative, on graded panels that exercise hot / cold /
frozen columns, the cold maintenance, refreshes and the blocked Q formation."""

import numpy as np
import pytest

from oracle import spand_oracle as orc
from tests.test_gpu_contract import assert_rrqr_matches, with_singular_values

pytestmark = pytest.mark.gpu


def _single(a, eps, scheme, cluster, group=None):
    from paper_2007_00789_b200.rrqr import rrqr_single
    return rrqr_single(a, eps, scheme, group=group, cluster=cluster)


def _graded(m, n, decades, seed):
    rng = np.random.default_rng(seed)
    svals = np.geomspace(1.0, 10.0 ** (-decades), min(m, n))
    a = with_singular_values(m, n, svals, seed=seed)
    # strongly varying column scales: most columns freeze, a few stay hot
    a *= np.geomspace(1.0, 1e-4, n)[rng.permutation(n)]
    return a + 1e-14 * rng.standard_normal((m, n))


@pytest.mark.parametrize("cluster", [2, 4, 8])
@pytest.mark.parametrize("m,n,eps,scheme,group", [
    (256, 1500, 1e-2, "second-full", None),
    (300, 2000, 1e-2, "second-superfine", 16),
    (520, 3000, 1e-2, "first", 24),
    (700, 4000, 1e-3, "second-full", 32),
    (1024, 6000, 1e-2, "second-full", 64),
])
def test_clustered_rrqr_matches_oracle(cluster, m, n, eps, scheme, group):
    a = _graded(m, n, 6, m + n)
    mine = _single(a, eps, scheme, cluster, group)
    ref = orc.sparsify_panel(a, eps, scheme)
    assert_rrqr_matches(mine, ref, tol=1e-10)


@pytest.mark.parametrize("scheme", ["first", "second-full", "second-superfine"])
def test_clustered_equals_classic_decisions(scheme):
    """Clustered and classic kernels take the same pivots on a tall panel
    with many groups (and agree on the payloads to rounding)."""
    a = _graded(1500, 9000, 8, 7)
    c = _single(a, 1e-2, scheme, 8, 128)
    k = _single(a, 1e-2, scheme, 0, 128)
    assert c.rank_c == k.rank_c and c.rank_f2 == k.rank_f2
    assert np.array_equal(np.asarray(c.perm), np.asarray(k.perm))
    for x, y in ((c.r_coarse, k.r_coarse), (c.q_c, k.q_c), (c.e_tilde, k.e_tilde)):
        assert x.shape == y.shape
        if y.size:
            assert np.linalg.norm(x - y) <= 1e-10 * max(1.0, np.linalg.norm(y))


def test_clustered_low_rank_and_zero_columns():
    """Exact low rank (every column frozen early), zero columns and a
    single-cluster group."""
    rng = np.random.default_rng(3)
    m, n, r = 400, 2500, 12
    a = (rng.standard_normal((m, r)) * np.geomspace(1.0, 1e-3, r)) @ rng.standard_normal((r, n))
    a[:, rng.choice(n, 300, replace=False)] = 0.0
    for scheme in ("first", "second-full", "second-superfine"):
        mine = _single(a, 1e-2, scheme, 8, 8)
        ref = orc.sparsify_panel(a, 1e-2, scheme)
        assert_rrqr_matches(mine, ref, tol=1e-10)


@pytest.mark.parametrize("tag", ["C4_L11_e0.01_second-full", "C3_L12_e0.01_second-full"])
def test_clustered_factorization_matches_reference(tag, monkeypatch):
    """Whole factorization with the large-panel waves clustered
    (SPAND_RRQR_CLUSTER=8): integer structure bit-exact against the
    reference's frozen outputs, n_cg within +-1 (tests/test_gpu_configs.py)."""
    from tests.golden_cases import hierarchy_for, load, matrix_for
    from tests.test_gpu_configs import sha
    import paper_2007_00789_b200 as sp
    monkeypatch.setenv("SPAND_RRQR_CLUSTER", "8")
    monkeypatch.setenv("SPAND_RRQR_CLUSTER_MIN", "128")
    rec, arr = load(tag)
    a = matrix_for(tag)
    h = hierarchy_for(tag, a, rec["levels"])
    f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"])
    got = [[[e["cluster"], e["size_before"], e["size_after"], e["rank_f2"]]
            for e in lv["interfaces"]] for lv in f.diagnostics["levels"]]
    assert got == [lv["interfaces"] for lv in rec["diagnostics"]]
    assert sha(np.asarray(f.perm, np.int64)) == rec["perm_sha"]
    _, rep = sp.pcg(a, arr["b"], m=f.apply_m, tol=rec["tol"])
    assert abs(rep.n_cg - rec["n_cg"]) <= 1
