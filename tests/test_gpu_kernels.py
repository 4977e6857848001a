"""Kernel-level parity on the B200 (reference test_dense.py style)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_spmv_matches_csr():
    from paper_2007_00789_b200 import baseline_problem
    a, b, _ = baseline_problem("C1")
    y = a.matvec(b)
    ref = a.to_scipy() @ b
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)


@pytest.mark.parametrize("n", [1, 5, 31, 32, 33, 63, 64, 65, 100, 257])
def test_cholesky_reconstruction(n):
    from paper_2007_00789_b200 import cholesky
    rng = np.random.default_rng(n)
    g = rng.standard_normal((n, n))
    m = g @ g.T + n * np.eye(n)
    l = cholesky(m)
    assert np.allclose(np.triu(l, 1), 0.0)
    assert np.linalg.norm(l @ l.T - m) / np.linalg.norm(m) <= 1e-13
    ref = np.linalg.cholesky(m)
    assert np.linalg.norm(l - ref) / np.linalg.norm(ref) <= 1e-13


def test_cholesky_hand_and_pivot():
    from paper_2007_00789_b200 import NotSPD, cholesky
    l = cholesky(np.array([[4.0, 2.0], [2.0, 5.0]]))
    assert np.allclose(l, [[2.0, 0.0], [1.0, 2.0]], atol=1e-15)
    with pytest.raises(NotSPD) as exc:
        cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert exc.value.pivot == 1
    with pytest.raises(NotSPD) as exc:
        cholesky(np.array([[-1.0]]))
    assert exc.value.pivot == 0
    # a failing pivot inside a block of <= 64 (the shared-memory path)
    g = np.random.default_rng(5).standard_normal((40, 40))
    m = g @ g.T + 40 * np.eye(40)
    m[23, 23] = -1e6
    with pytest.raises(NotSPD) as exc:
        cholesky(m)
    assert exc.value.pivot == 23
    rng = np.random.default_rng(3)
    g = rng.standard_normal((70, 70))
    m = g @ g.T + 70 * np.eye(70)
    m[50, 50] = -1e6
    with pytest.raises(NotSPD) as exc:
        cholesky(m)
    from oracle.spand_oracle import OracleNotSPD, chol
    with pytest.raises(OracleNotSPD) as ref:
        chol(m)
    assert exc.value.pivot == ref.value.pivot


@pytest.mark.parametrize("n", [1, 8, 40, 63, 64, 130])
def test_tri_inverse(n):
    from paper_2007_00789_b200 import tri_inverse
    rng = np.random.default_rng(2)
    l = np.tril(rng.standard_normal((n, n))) + 4.0 * np.eye(n)
    assert np.allclose(tri_inverse(l) @ l, np.eye(n), atol=1e-12)


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("side", ["left", "right"])
def test_tri_solve_residual(trans, side):
    from paper_2007_00789_b200 import tri_solve
    rng = np.random.default_rng(1)
    l = np.tril(rng.standard_normal((25, 25))) + 5.0 * np.eye(25)
    b = rng.standard_normal((25, 3)) if side == "left" else rng.standard_normal((3, 25))
    x = tri_solve(l, b, trans=trans, side=side)
    op = l.T if trans else l
    lhs = op @ x if side == "left" else x @ op
    assert np.linalg.norm(lhs - b) / np.linalg.norm(b) <= 1e-13


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (64, 16, 64), (65, 17, 63),
                                   (200, 300, 130), (7, 1000, 5)])
@pytest.mark.parametrize("tb", [False, True])
def test_gemm_dmma(m, k, n, tb):
    from paper_2007_00789_b200.kernels import gemm_one
    rng = np.random.default_rng(m + k + n)
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((n, k)) if tb else rng.standard_normal((k, n))
    c = gemm_one(a, b, trans_b=tb)
    ref = a @ (b.T if tb else b)
    assert np.linalg.norm(c - ref) <= 1e-13 * max(1.0, np.linalg.norm(ref))
