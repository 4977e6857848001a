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
