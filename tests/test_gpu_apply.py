"""Device apply + PCG on factors frozen from the reference (SPDF files).

The reference's own factor is loaded onto the B200 and applied with the
batched plan; apply_m must match the reference's apply_m to rounding and
PCG must take exactly the reference's iteration count.
"""

import glob
import os

import numpy as np
import pytest

from tests.golden_cases import GOLDEN, load, matrix_for

pytestmark = pytest.mark.gpu

SPDF = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLDEN, "*.spdf")))


@pytest.mark.parametrize("tag", SPDF)
def test_loaded_reference_factor_applies(tag):
    from paper_2007_00789_b200 import load_factor, pcg
    rec, arr = load(tag)
    f = load_factor(os.path.join(GOLDEN, tag + ".spdf"))
    assert f.nnz_factor == rec["nnz_factor"]
    z = f.apply_m(arr["b"])
    ref = arr["apply_m_b"]
    assert np.linalg.norm(z - ref) <= 1e-12 * np.linalg.norm(ref)
    a = matrix_for(tag)
    x, rep = pcg(a, arr["b"], m=f.apply_m, tol=rec["tol"])
    assert rep.n_cg == rec["n_cg"]
    np.testing.assert_allclose(rep.residual_history, rec["residual_history"],
                               rtol=1e-6, atol=1e-15)
    # apply_inv_t is the transpose of apply_inv
    n = f.n
    if n <= 300:
        li = np.column_stack([f.apply_inv(c) for c in np.eye(n)])
        lt = np.column_stack([f.apply_inv_t(c) for c in np.eye(n)])
        assert np.allclose(lt, li.T, atol=1e-13)
    # column stacks
    stack = np.column_stack([arr["b"], 2 * arr["b"]])
    zz = f.apply_m(stack)
    assert np.allclose(zz[:, 0], z, rtol=0, atol=1e-13 * np.abs(z).max())
    assert np.allclose(zz[:, 1], 2 * z, rtol=0, atol=1e-13 * np.abs(z).max())


@pytest.mark.gpu
@pytest.mark.parametrize("case", [("lap3d", 16, 6), ("hc3d", 16, 7)])
def test_row_compressed_image_is_bitwise_identical(case, monkeypatch):
    """The first apply image keeps every elimination-panel row; the
    row-compressed image (device nonzero-row bits, compiled in the
    background) replaces it later.  Both must give the same bits for
    apply_m, apply_inv, apply_inv_t and column stacks (fastplan.py,
    collect.cpp compile_phase: fixed summation groups)."""
    import paper_2007_00789_b200 as sp
    from paper_2007_00789_b200.fastplan import NativeApplyPlan
    kind, d, lv = case
    a = sp.laplacian_3d(d) if kind == "lap3d" else sp.baseline_problem("C4", grid=d)[0]
    h = sp.build_hierarchy(a, lv)
    b = np.random.default_rng(1).standard_normal((a.n, 3))

    def results(f):
        return [f.apply_m(b[:, 0]), f.apply_inv(b[:, 1]), f.apply_inv_t(b[:, 2]), f.apply_m(b)]
    monkeypatch.setattr(NativeApplyPlan, "ROW_COMPRESS", False)
    f1 = sp.factorize(a, h, 0.01, "second-full", skip_levels=2)
    plain = results(f1)
    assert "compressed" not in f1.plan.build_times
    monkeypatch.setattr(NativeApplyPlan, "ROW_COMPRESS", True)
    f2 = sp.factorize(a, h, 0.01, "second-full", skip_levels=2)
    f2.apply_m(b[:, 0])
    if f2.plan._future2 is not None:
        f2.plan._future2.result()
    comp = results(f2)
    assert f2.plan.build_times.get("compressed") is not None
    for x, y in zip(plain, comp):
        assert np.array_equal(x, y)
