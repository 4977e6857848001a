"""Multi-RHS apply of engine factors (the reference's
apply_* accept an n x k column stack, factorize.py:262-267).

The device path pushes up to 8 vectors through one pass of the factor
(payload read once per group of 4): every column must equal the
single-vector apply bit for bit (same per-vector summation order), and the
stack must match the oracle's apply_m."""

import numpy as np
import pytest

import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2, 3, 5, 9])
def test_multirhs_apply_matches_columns(k):
    a = sp.laplacian_3d(12)
    h = sp.build_hierarchy(a, 6)
    f = sp.factorize(a, h, 0.01, "second-full", skip_levels=2)
    rng = np.random.default_rng(k)
    x = rng.standard_normal((a.n, k))
    zs = f.apply_m(x)
    assert zs.shape == (a.n, k)
    for j in range(k):
        assert np.array_equal(zs[:, j], f.apply_m(x[:, j]))
    for fn in ("apply_inv", "apply_inv_t"):
        zz = getattr(f, fn)(x)
        for j in range(k):
            assert np.array_equal(zz[:, j], getattr(f, fn)(x[:, j]))
    cl = orc.nd_hierarchy(a.n, a.row_ptr, a.col_idx, 6)
    of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, 6, 0.01, "second-full", 2)
    zr = of.apply_m(x)
    assert np.linalg.norm(zs - zr) <= 1e-9 * np.linalg.norm(zr)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 3, 6])
def test_pcg_multi_matches_single_bitwise(k):
    """Multi-RHS PCG: every column's solution, residual
    history, n_cg and stopping decision are bit for bit those of the
    single-vector pcg (same kernels, same order; the stacked preconditioner
    apply is bitwise per column); a zero column returns immediately."""
    import paper_2007_00789_b200 as sp
    a, _, lv = sp.baseline_problem("C1")
    h = sp.build_hierarchy(a, lv)
    f = sp.factorize(a, h, 0.01, "second-full")
    rng = np.random.default_rng(k)
    bs = rng.standard_normal((a.n, k))
    if k > 1:
        bs[:, 1] = 0.0
    x, reps = sp.pcg(a, bs, m=f.apply_m, tol=1e-12)
    assert x.shape == (a.n, k) and len(reps) == k
    for j in range(k):
        if not np.any(bs[:, j]):
            assert reps[j].n_cg == 0 and np.all(x[:, j] == 0.0)
            continue
        xs, rs = sp.pcg(a, bs[:, j], m=f.apply_m, tol=1e-12)
        assert np.array_equal(x[:, j], xs)
        assert reps[j].residual_history == rs.residual_history
        assert reps[j].n_cg == rs.n_cg and reps[j].converged == rs.converged
        assert reps[j].true_residual == rs.true_residual
