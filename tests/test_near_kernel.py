"""Near-kernel preservation (EXTENSION).

The reference has no near-kernel mode (SPEC.md:350 lists it as a non-goal;
PAPER.md:2005 names it as compatible future work), so its oracle is the CPU
restatement ``oracle.spand_oracle.sparsify_panel_nk``, pinned here by
known-answer properties:

- with no vectors (None, or k = 0, or all-zero vectors) the factorization is
  the reference path BITWISE (fixture payload hashes of the golden cases);
- ``nk_basis`` is a Householder QR: H orthogonal, H^T u = [R_u; 0], the rank
  drops for dependent vectors;
- each nk sparsification is an orthogonal change of basis of the panel:
  q^T W = [e_tilde rows; r_coarse rows] and span(u_p) lies in span(q_c);
- on a matrix with a nearly exact kernel (Neumann Laplacian + 1e-8 I) the
  preconditioner becomes exact on that kernel: ||(I - M A) 1|| / ||1|| drops
  from O(1) to < 1e-5 and PCG needs fewer iterations.

GPU tests (-m gpu) check the device path against this oracle: interface
ranks bit-exact, perm equal, apply_m within 1e-9, n_cg equal.
"""

import numpy as np
import pytest
import scipy.sparse as sps

import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc
from paper_2007_00789_b200.errors import DimensionMismatch
from tests.golden_cases import load, matrix_for


def _neumann(a, shift):
    """Graph Laplacian of a's off-diagonal pattern (rows sum to shift)."""
    m = sps.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    off = m - sps.diags(m.diagonal())
    d = -np.asarray(off.sum(axis=1)).ravel() + shift
    b = (off + sps.diags(d)).tocsr()
    b.sort_indices()
    return sp.SparseSymMatrix(a.n, b.indptr.astype(np.int64), b.indices.astype(np.int64),
                              b.data.astype(np.float64))


def _oracle(a, levels, eps, scheme, skip, nk):
    cl = orc.nd_hierarchy(a.n, a.row_ptr, a.col_idx, levels)
    f = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, levels, eps, scheme, skip,
                      near_kernel=nk)
    return cl, f


def test_nk_basis_is_householder_qr():
    rng = np.random.default_rng(5)
    u = rng.standard_normal((40, 4))
    u[:, 3] = u[:, 0] - 2.0 * u[:, 1]          # dependent column
    vs, taus, ru = orc.nk_basis(u)
    assert len(vs) == 3
    h = orc.nk_explicit(vs, taus, 40)
    assert np.allclose(h.T @ h, np.eye(40), atol=1e-13)
    hu = h.T @ u
    assert np.allclose(hu[:3], ru, atol=1e-12)
    assert np.linalg.norm(hu[3:]) <= 1e-12 * np.linalg.norm(u)
    assert np.allclose(orc.nk_reflect(vs, taus, u), hu, atol=1e-12)
    # zero vectors: no reflectors
    vs0, _, ru0 = orc.nk_basis(np.zeros((10, 2)))
    assert vs0 == [] and ru0.shape == (0, 2)


@pytest.mark.parametrize("scheme", ["first", "second-full", "second-superfine"])
def test_sparsify_panel_nk_is_orthogonal_change_of_basis(scheme):
    rng = np.random.default_rng(7)
    m, n = 30, 50
    w = rng.standard_normal((m, 8)) @ rng.standard_normal((8, n))
    w += 1e-3 * rng.standard_normal((m, n))
    u = np.column_stack([np.ones(m), np.arange(m, dtype=float)])
    res, r, ru = orc.sparsify_panel_nk(w, u, 0.05, scheme)
    assert r == 2
    q = np.hstack([res["q_f"], res["q_c"]])
    assert np.allclose(q.T @ q, np.eye(m), atol=1e-12)
    kc = res["rank_c"]
    qtw = q.T @ w
    assert np.allclose(qtw[m - kc:], res["r_coarse"], atol=1e-11)
    ne = res["e_tilde"].shape[0]
    if ne:
        assert np.allclose(qtw[:ne], res["e_tilde"], atol=1e-11)
    # span(u) inside span(q_c): no fine component
    assert np.linalg.norm(res["q_f"].T @ u) <= 1e-12 * np.linalg.norm(u)
    # the last r coarse columns are U, with U^T u = R_u
    assert np.allclose(res["q_c"][:, kc - r:].T @ u, ru, atol=1e-12)


def test_no_vectors_is_reference_path_bitwise():
    """None, k = 0 and all-zero vectors all give the reference factor."""
    tag = "lap2d_d16_L4_e0.05_k1_second-full"
    meta = load(tag)[0]
    a = matrix_for(tag)
    levels, eps, scheme, skip = meta["levels"], meta["eps"], meta["scheme"], meta["skip_levels"]
    _, f0 = _oracle(a, levels, eps, scheme, skip, None)
    for nk in (np.zeros((a.n, 0)), np.zeros(a.n), np.zeros((a.n, 3))):
        _, f1 = _oracle(a, levels, eps, scheme, skip, nk)
        assert len(f1.ops) == len(f0.ops)
        for o0, o1 in zip(f0.ops, f1.ops):
            assert o0.kind == o1.kind
            assert np.array_equal(o0.dofs, o1.dofs)
            for name in ("lower", "panel", "q", "e_tilde"):
                x0, x1 = getattr(o0, name), getattr(o1, name)
                if x0 is not None:
                    assert np.array_equal(x0, x1), name
        assert np.array_equal(f0.perm, f1.perm)


@pytest.mark.parametrize("grid,levels", [("2d", 8), ("3d", 8)])
@pytest.mark.parametrize("scheme", ["first", "second-full"])
def test_exact_kernel_is_preserved(grid, levels, scheme):
    a0 = sp.laplacian_2d(64) if grid == "2d" else sp.laplacian_3d(16)
    a = _neumann(a0, 1e-8)
    mv = orc.csr_matvec(a.n, a.row_ptr, a.col_idx, a.values)
    ones = np.ones(a.n)
    b = np.random.default_rng(0).standard_normal(a.n)
    out = {}
    for key, nk in (("off", None), ("on", ones)):
        _, f = _oracle(a, levels, 0.1, scheme, 2, nk)
        fe = np.linalg.norm(ones - f.apply_m(mv(ones))) / np.linalg.norm(ones)
        _, its, *_ = orc.pcg(mv, b, f.apply_m, 1e-10)
        out[key] = (fe, its)
    assert out["off"][0] > 0.5
    assert out["on"][0] < 1e-5
    assert out["on"][1] < out["off"][1]


def test_near_kernel_argument_errors():
    a = sp.laplacian_2d(8)
    h = sp.build_hierarchy(a, 3)
    with pytest.raises(DimensionMismatch):
        sp.factorize(a, h, 0.1, "first", near_kernel=np.ones(a.n + 1))
    with pytest.raises(ValueError):
        sp.factorize(a, h, 0.1, "first", near_kernel=np.ones((a.n, 17)))


# ---------------------------------------------------------------- device


def _vectors(a, kind):
    n = a.n
    if kind == "ones":
        return np.ones(n)
    d = int(round(n ** 0.5))
    x, y = np.meshgrid(np.arange(d, dtype=float), np.arange(d, dtype=float), indexing="ij")
    return np.column_stack([np.ones(n), x.ravel() / d, y.ravel() / d])


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    ("lap2d", 32, 5, 0.01, "second-full", 1, "ones"),
    ("lap2d", 32, 5, 0.01, "first", 1, "ones"),
    ("lap2d", 32, 5, 0.05, "second-superfine", 1, "ones"),
    ("lap2d", 48, 6, 0.05, "second-full", 2, "linear"),
    ("neu2d", 48, 6, 0.1, "second-full", 2, "ones"),
    ("lap3d", 12, 6, 0.01, "second-full", 2, "ones"),
])
def test_device_near_kernel_matches_oracle(case):
    kind, d, levels, eps, scheme, skip, vec = case
    if kind == "lap3d":
        a = sp.laplacian_3d(d)
    else:
        a = sp.laplacian_2d(d)
        if kind == "neu2d":
            a = _neumann(a, 1e-8)
    nk = _vectors(a, vec)
    b = np.random.default_rng(1).standard_normal(a.n)
    h = sp.build_hierarchy(a, levels)
    f = sp.factorize(a, h, eps, scheme, skip_levels=skip, near_kernel=nk)
    cl, of = _oracle(a, levels, eps, scheme, skip, nk)
    got = [[(e["cluster"], e["size_before"], e["size_after"], e["rank_f2"])
            for e in lv["interfaces"]] for lv in f.diagnostics["levels"]]
    want = [[tuple(e) for e in lv["interfaces"]] for lv in of.diagnostics["levels"]]
    assert got == want
    assert np.array_equal(f.perm, of.perm)
    z, zr = f.apply_m(b), of.apply_m(b)
    # neu2d: cond(A) ~ 1e8 (kernel shift 1e-8), so M b is dominated by the
    # kernel component and rounding is amplified accordingly
    tol = 1e-7 if kind == "neu2d" else 1e-9
    assert np.linalg.norm(z - zr) <= tol * np.linalg.norm(zr)
    mv = orc.csr_matvec(a.n, a.row_ptr, a.col_idx, a.values)
    _, its, *_ = orc.pcg(mv, b, of.apply_m, 1e-12)
    _, rep = sp.pcg(a, b, m=f.apply_m, tol=1e-12)
    assert abs(rep.n_cg - its) <= 1
    # the device factor is also exact on the preserved kernel
    if kind == "neu2d":
        ones = np.ones(a.n)
        fe = np.linalg.norm(ones - f.apply_m(mv(ones))) / np.linalg.norm(ones)
        assert fe < 1e-5
