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
