"""Input side on the device (reference sparse.py:181-308):
the finite-volume generator of the BASELINE configs and the Jacobi prescale
run on the B200 (csrc/input.cu) and give the host generator's matrices bit
for bit, with the device CSR left cached on the matrix."""

import numpy as np
import pytest

import paper_2007_00789_b200 as sp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,grid", [("C1", None), ("C2", None), ("C3", 64), ("C4", None),
                                       ("C3", None)])
def test_device_generator_matches_host(name, grid):
    a, b, lv = sp.baseline_problem(name, grid=grid)
    d, bd, lvd = sp.baseline_problem(name, grid=grid, device=True)
    assert lv == lvd and np.array_equal(b, bd)
    assert d.n == a.n
    assert np.array_equal(d.row_ptr, a.row_ptr)
    assert np.array_equal(d.col_idx, a.col_idx)
    assert np.array_equal(d.values, a.values)
    # the cached device CSR is the one the SpMV uses (no upload)
    assert None in d._dev
    x = np.random.default_rng(0).standard_normal(a.n)
    assert np.array_equal(d.matvec(x), a.matvec(x))


def test_device_generator_rejects_bad_shapes():
    with pytest.raises(sp.DimensionMismatch):
        sp.diffusion_fv_device(np.ones((3, 3)), 4, (10, 12))
    with pytest.raises(sp.NonpositiveDiagonal):
        sp.diffusion_fv_device(-np.ones((2, 2)), 4, (8, 8))


@pytest.mark.parametrize("name", ["C1", "C4"])
def test_device_jacobi_prescale_matches_host(name):
    a, b, _ = sp.baseline_problem(name)
    s1, b1, d1 = sp.jacobi_prescale(a, b)
    s2, b2, d2 = sp.jacobi_prescale(a, b, device=True)
    assert np.array_equal(s1.values, s2.values)
    assert np.array_equal(b1, b2) and np.array_equal(d1, d2)
    assert np.array_equal(s1.col_idx, s2.col_idx)


def test_device_jacobi_prescale_rejects_nonpositive_diagonal():
    a = sp.laplacian_2d(6)
    vals = a.values.copy()
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    vals[(rows == a.col_idx) & (rows == 7)] = 1e-300
    z = sp.SparseSymMatrix(a.n, a.row_ptr, a.col_idx, vals)
    s, _, _ = sp.jacobi_prescale(z, np.ones(a.n), device=True)   # tiny but positive
    assert np.all(np.isfinite(s.values))
