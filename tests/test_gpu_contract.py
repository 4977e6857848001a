"""The reference's hot-path contract tests, restated against the device path.

Each test follows a reference test (cited) and, where the reference test
only checks a property, also compares with the CPU oracle on the same
input:

- RRQR semantics (pkg/tests/test_dense.py:117-257) through the public
  ``rrqr_sparsify`` (the device RRQR wave kernel): identical perm, rank_c,
  rank_f2 as the oracle, payloads within 1e-12;
- bitwise determinism of a factorization (test_factorize.py:173-186);
- first-order vs second-full base operators bitwise equal
  (test_factorize.py:116-137);
- per-level trailing-matrix digests identical across schemes
  (test_factorize.py:104-113);
- SPDF round trip (test_factorize.py:279-330): our file read back by our
  loader AND by the oracle's independent reader (factorize.py:452-502);
- two factorizations, then the first one applied (each factor owns its
  apply image);
- the e_tilde sign-flip fault injection of test_cli.py:265-281 against the
  device factor (the second-order quality guard of cli.py:512-563 trips).
"""

import hashlib

import numpy as np
import pytest

from oracle import spand_oracle as orc

pytestmark = pytest.mark.gpu

ALL_SCHEMES = ["first", "second-full", "second-superfine"]


def _sp():
    import paper_2007_00789_b200 as sp
    return sp


def with_singular_values(m, n, svals, seed=0):
    """Random matrix with prescribed singular values (test_dense.py:23-31)."""
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.zeros((m, n))
    k = min(len(svals), m, n)
    s[:k, :k] = np.diag(svals[:k])
    return u @ s @ v.T


def rrqr_both(a, eps, scheme):
    sp = _sp()
    mine = sp.rrqr_sparsify(a, eps, scheme)
    ref = orc.sparsify_panel(a, eps, scheme)
    return mine, ref


def assert_rrqr_matches(mine, ref, tol=1e-12):
    """Integer decisions identical, payloads within tol (relative)."""
    assert mine.rank_c == ref["rank_c"]
    assert mine.rank_f2 == ref["rank_f2"]
    kstop = ref["k_stop"]
    assert np.array_equal(np.asarray(mine.perm)[:kstop], ref["perm"][:kstop])
    for got, want in ((mine.q_c, ref["q_c"]), (mine.r_coarse, ref["r_coarse"]),
                      (mine.e_tilde, ref["e_tilde"])):
        assert got.shape == want.shape
        if want.size:
            scale = max(1.0, np.linalg.norm(want))
            assert np.linalg.norm(got - want) <= tol * scale
    # q_f is unique only up to the span of its noise-level columns
    assert mine.q_f.shape == ref["q_f"].shape
    if ref["q_f"].size:
        pa = mine.q_f @ mine.q_f.T
        pb = ref["q_f"] @ ref["q_f"].T
        assert np.linalg.norm(pa - pb) <= tol * max(1.0, np.linalg.norm(pb))


# ---------------------------------------------------------------------------
# RRQR (test_dense.py:117-257)


@pytest.mark.parametrize("scheme", ALL_SCHEMES)
def test_rrqr_zero_panel(scheme):
    sp = _sp()
    res = sp.rrqr_sparsify(np.zeros((5, 8)), 0.1, scheme)
    assert res.rank_c == 0
    assert np.array_equal(res.q_f, np.eye(5))
    assert res.q_c.shape == (5, 0)
    assert res.r_coarse.shape == (0, 8)
    if scheme == "second-full":
        assert res.e_tilde.shape == (5, 8)
        assert np.array_equal(res.e_tilde, np.zeros((5, 8)))


def test_rrqr_diagonal_pivots_first_order():
    a = np.zeros((2, 4))
    a[0, 0] = 1.0
    a[1, 1] = 1e-3
    mine, ref = rrqr_both(a, 0.1, "first")
    assert mine.rank_c == 1
    assert mine.e_tilde.shape == (0, 4)
    assert abs(np.linalg.norm(mine.q_f.T @ a, 2) - 1e-3) <= 1e-18
    assert_rrqr_matches(mine, ref)


def test_rrqr_superfine_ranks_match_svd_counts():
    svals = np.array([10.0 ** -k for k in range(12)])
    a = with_singular_values(12, 20, svals, seed=3)
    mine, ref = rrqr_both(a, 1e-3, "second-superfine")
    sv = np.linalg.svd(a, compute_uv=False)
    assert abs(mine.rank_c - int(np.sum(sv >= 1e-3))) <= 1
    assert abs(mine.rank_f2 - int(np.sum((sv >= 1e-6) & (sv < 1e-3)))) <= 1
    assert_rrqr_matches(mine, ref)


@pytest.mark.parametrize("shape", [(12, 20), (20, 12)])
def test_rrqr_exact_reconstruction_at_zero_eps(shape):
    a = np.random.default_rng(4).standard_normal(shape)
    mine, ref = rrqr_both(a, 0.0, "second-full")
    q = np.hstack([mine.q_c, mine.q_f])
    r = np.vstack([mine.r_coarse, mine.e_tilde])
    assert np.linalg.norm(q @ r - a) / np.linalg.norm(a) <= 1e-12
    assert mine.rank_c == ref["rank_c"] == min(shape)


@pytest.mark.parametrize("scheme", ALL_SCHEMES)
@pytest.mark.parametrize("seed,shape,eps", [
    (0, (10, 16), 0.1), (1, (16, 10), 1e-2), (2, (9, 9), 1e-4),
    (3, (6, 30), 0.5), (4, (30, 6), 1e-6), (5, (13, 13), 0.0),
])
def test_rrqr_orthogonality_and_partition(scheme, seed, shape, eps):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(shape) * np.exp(rng.standard_normal(shape))
    mine, ref = rrqr_both(a, eps, scheme)
    q = np.hstack([mine.q_c, mine.q_f])
    m = shape[0]
    assert q.shape == (m, m)
    assert np.linalg.norm(q.T @ q - np.eye(m)) <= 1e-12
    assert mine.rank_c + mine.q_f.shape[1] == m
    assert np.allclose(mine.r_coarse, mine.q_c.T @ a, atol=1e-12)
    assert_rrqr_matches(mine, ref)


def test_rrqr_full_scheme_correction_is_fine_projection():
    a = np.random.default_rng(6).standard_normal((8, 14))
    mine, ref = rrqr_both(a, 0.05, "second-full")
    assert np.allclose(mine.e_tilde, mine.q_f.T @ a, atol=1e-12)
    assert_rrqr_matches(mine, ref)


def test_rrqr_rank_nonincreasing_in_eps():
    sp = _sp()
    a = with_singular_values(11, 18, np.geomspace(1.0, 1e-10, 11), seed=7)
    ranks = []
    for eps in (0.0, 1e-8, 1e-6, 1e-4, 1e-2, 0.5, 1.0):
        res = sp.rrqr_sparsify(a, eps, "first")
        assert res.rank_c == orc.sparsify_panel(a, eps, "first")["rank_c"]
        ranks.append(res.rank_c)
    assert all(r1 >= r2 for r1, r2 in zip(ranks, ranks[1:]))
    assert ranks[0] == 11


@pytest.mark.parametrize("seed", range(6))
def test_rrqr_dropped_norm_bound(seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((12, 19)) * np.exp(2 * rng.standard_normal((12, 19)))
    mine, ref = rrqr_both(a, 1e-2, "second-full")
    r11 = np.max(np.linalg.norm(a, axis=0))
    dropped = np.linalg.norm(mine.q_f.T @ a, 2) if mine.q_f.size else 0.0
    assert dropped <= r11 * 1e-2 * np.sqrt(19)
    assert_rrqr_matches(mine, ref)


def test_rrqr_superfine_with_empty_band_equals_first_order():
    sp = _sp()
    a = with_singular_values(5, 9, [1.0, 0.5, 0.2, 1e-8, 1e-9], seed=8)
    fo = sp.rrqr_sparsify(a, 1e-3, "first")
    sf = sp.rrqr_sparsify(a, 1e-3, "second-superfine")
    assert sf.rank_f2 == 0
    assert sf.rank_c == fo.rank_c
    assert np.array_equal(sf.q_c, fo.q_c)
    assert np.array_equal(sf.r_coarse, fo.r_coarse)
    assert sf.e_tilde.shape[0] == 0


def test_rrqr_superfine_with_full_band_matches_full_scheme():
    sp = _sp()
    a = with_singular_values(5, 11, [1.0, 0.5, 1e-4, 5e-5, 2e-5], seed=9)
    full = sp.rrqr_sparsify(a, 1e-3, "second-full")
    sf = sp.rrqr_sparsify(a, 1e-3, "second-superfine")
    assert sf.rank_c == full.rank_c
    assert sf.rank_f2 == 5 - sf.rank_c
    assert np.array_equal(sf.q_c, full.q_c)
    assert np.array_equal(sf.r_coarse, full.r_coarse)
    assert np.allclose(full.e_tilde.T @ full.e_tilde, sf.e_tilde.T @ sf.e_tilde, atol=1e-12)


def test_rrqr_full_rank_panel_is_noop():
    sp = _sp()
    rng = np.random.default_rng(10)
    q, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    a = q @ np.diag([3.0, 2.5, 2.0, 1.5, 1.2, 1.0]) @ q.T
    res = sp.rrqr_sparsify(a, 1e-6, "first")
    assert res.rank_c == 6
    assert res.q_f.shape == (6, 0)


def test_rrqr_rejects_bad_input():
    sp = _sp()
    a = np.ones((3, 3))
    a[1, 2] = np.nan
    with pytest.raises(sp.NonFinite):
        sp.rrqr_sparsify(a, 0.1, "first")
    with pytest.raises(ValueError):
        sp.rrqr_sparsify(np.ones((2, 2)), 1.5, "first")
    with pytest.raises(ValueError):
        sp.rrqr_sparsify(np.ones((2, 2)), -0.1, "first")


def test_rrqr_empty_panels():
    sp = _sp()
    res = sp.rrqr_sparsify(np.zeros((0, 5)), 0.1, "first")
    assert res.rank_c == 0 and res.q_f.shape == (0, 0)
    res = sp.rrqr_sparsify(np.zeros((4, 0)), 0.1, "second-full")
    assert res.rank_c == 0 and np.array_equal(res.q_f, np.eye(4))


@pytest.mark.parametrize("m,n,eps,scheme", [
    (300, 2000, 1e-2, "second-full"), (700, 5000, 1e-2, "second-superfine"),
    (1100, 9000, 1e-3, "first")])
def test_rrqr_stress_panels_match_oracle(m, n, eps, scheme):
    """Multi-CTA groups, cold / frozen columns and the blocked Q formation
     on graded panels, decisions identical to the oracle."""
    rng = np.random.default_rng(m + n)
    svals = np.geomspace(1.0, 1e-9, min(m, n))
    a = with_singular_values(m, n, svals, seed=m)
    a += 1e-14 * rng.standard_normal((m, n))
    mine, ref = rrqr_both(a, eps, scheme)
    assert_rrqr_matches(mine, ref, tol=1e-10)


def test_rrqr_panel_taller_than_6144_rows():
    """Panels above the round-1 6144-row limit (the reference has none):
    a 7000 x 7400 panel of numerical rank ~24 against the oracle."""
    rng = np.random.default_rng(12)
    m, n, r = 7000, 7400, 24
    a = (rng.standard_normal((m, r)) * np.geomspace(1.0, 1e-3, r)) @ rng.standard_normal((r, n))
    a += 1e-9 * rng.standard_normal((m, n))
    mine, ref = rrqr_both(a, 1e-2, "second-superfine")
    assert_rrqr_matches(mine, ref, tol=1e-10)


# ---------------------------------------------------------------------------
# factorization contract (test_factorize.py)


def _payloads(op):
    out = {}
    for name in ("lower", "panel", "q", "e_tilde"):
        if hasattr(op, name):
            out[name] = np.asarray(getattr(op, name))
    return out


@pytest.mark.parametrize("case", ["lap2d16", "hc3d16", "C1"])
def test_factorization_is_deterministic(case):
    """test_factorize.py:173-186, plus a 3D high-contrast case whose RRQR
    panels run on multi-CTA groups with atomic column lists, and C1."""
    sp = _sp()
    if case == "lap2d16":
        a, lv, eps, scheme, skip = sp.laplacian_2d(16), 4, 0.05, "second-full", 1
    elif case == "hc3d16":
        r = np.random.default_rng(3)
        a = sp.diffusion_fv(sp.log_uniform_block_field((16, 16, 16), 4, 3.0, r))
        lv, eps, scheme, skip = 8, 0.01, "second-full", 2
    else:
        a, _, lv = sp.baseline_problem("C1")
        eps, scheme, skip = 0.01, "second-superfine", 4
    h = sp.build_hierarchy(a, lv)
    fa = sp.factorize(a, h, eps, scheme, skip_levels=skip)
    fb = sp.factorize(a, h, eps, scheme, skip_levels=skip)
    assert len(fa.ops) == len(fb.ops)
    assert np.array_equal(fa.perm, fb.perm)
    assert fa.nnz_factor == fb.nnz_factor
    for x, y in zip(fa.ops, fb.ops):
        assert x.kind is y.kind
        assert np.array_equal(x.dofs, y.dofs)
        px, py = _payloads(x), _payloads(y)
        for name in px:
            assert np.array_equal(px[name], py[name]), (x.kind, name)
    b = np.random.default_rng(1).standard_normal(a.n)
    assert np.array_equal(fa.apply_m(b), fb.apply_m(b))
    assert [lv_["digest"] for lv_ in fa.diagnostics["levels"]] == \
        [lv_["digest"] for lv_ in fb.diagnostics["levels"]]


def test_factors_differ_only_by_corrections():
    """test_factorize.py:116-137 on the device path."""
    sp = _sp()
    a = sp.laplacian_2d(64)
    h = sp.build_hierarchy(a, sp.default_levels(a.n))
    fo = sp.factorize(a, h, 0.01, "first")
    fu = sp.factorize(a, h, 0.01, "second-full")
    fu_base = [op for op in fu.ops if op.kind is not sp.OpKind.ERROR_CORRECTION]
    assert all(op.kind is not sp.OpKind.ERROR_CORRECTION for op in fo.ops)
    assert any(op.kind is sp.OpKind.ERROR_CORRECTION for op in fu.ops)
    assert len(fo.ops) == len(fu_base)
    for x, y in zip(fo.ops, fu_base):
        assert x.kind is y.kind
        assert np.array_equal(x.dofs, y.dofs)
        px, py = _payloads(x), _payloads(y)
        assert px.keys() == py.keys()
        for name in px:
            assert np.array_equal(px[name], py[name]), (x.kind, name)


def test_trailing_matrices_identical_across_schemes():
    """test_factorize.py:104-113: the per-level trailing-matrix digests do
    not depend on the scheme; they do depend on eps (a changed trailing
    matrix changes the fingerprint)."""
    sp = _sp()
    a = sp.laplacian_2d(64)
    h = sp.build_hierarchy(a, sp.default_levels(a.n))
    dig = {}
    for s in ALL_SCHEMES:
        f = sp.factorize(a, h, 0.01, s)
        dig[s] = [lv["digest"] for lv in f.diagnostics["levels"]]
        assert all(isinstance(d, str) and len(d) == 64 for d in dig[s])
    assert dig["first"] == dig["second-full"]
    assert dig["first"] == dig["second-superfine"]
    other = sp.factorize(a, h, 0.1, "first")
    odig = [lv["digest"] for lv in other.diagnostics["levels"]]
    skipped = [lv["skipped"] for lv in other.diagnostics["levels"]]
    # levels inside the skip window see the same (exact) trailing matrix;
    # an empty trailing matrix (after the last level) hashes the same
    empty = hashlib.sha256(b"").hexdigest()
    for d0, d1, sk in zip(dig["first"], odig, skipped):
        if d0 != empty:
            assert (d0 == d1) == sk
    off = sp.factorize(a, h, 0.01, "first", digest=False)
    assert all(lv["digest"] is None for lv in off.diagnostics["levels"])


def test_two_factorizations_then_apply_first():
    """Each factor owns its apply image: factor A, factor B, then apply A
    (a shared staging buffer let B's image replace A's)."""
    sp = _sp()
    r = np.random.default_rng(3)
    a1 = sp.diffusion_fv(sp.log_uniform_block_field((16, 16, 16), 4, 3.0, r))
    h1 = sp.build_hierarchy(a1, 8)
    a2 = sp.laplacian_2d(96)
    h2 = sp.build_hierarchy(a2, 9)
    f1 = sp.factorize(a1, h1, 0.01, "second-full", skip_levels=2)
    f2 = sp.factorize(a2, h2, 0.01, "first")
    b1 = np.random.default_rng(5).standard_normal(a1.n)
    b2 = np.random.default_rng(6).standard_normal(a2.n)
    z1 = f1.apply_m(b1)
    z2 = f2.apply_m(b2)
    cl1 = [(c.id, c.dofs, c.depth) for c in h1.clusters]
    o1 = orc.factorize(a1.n, a1.row_ptr, a1.col_idx, a1.values, cl1, 8, 0.01,
                       "second-full", 2)
    ref1 = o1.apply_m(b1)
    assert np.linalg.norm(z1 - ref1) <= 1e-9 * np.linalg.norm(ref1)
    cl2 = [(c.id, c.dofs, c.depth) for c in h2.clusters]
    o2 = orc.factorize(a2.n, a2.row_ptr, a2.col_idx, a2.values, cl2, 9, 0.01, "first", 4)
    ref2 = o2.apply_m(b2)
    assert np.linalg.norm(z2 - ref2) <= 1e-9 * np.linalg.norm(ref2)


@pytest.mark.parametrize("scheme", ALL_SCHEMES)
def test_save_factor_round_trip(tmp_path, scheme):
    """test_factorize.py:279-330: a device-written SPDF file is read back
    (a) by load_factor with every field and payload bitwise equal and the
    same preconditioner, and (b) by the oracle's independent reader
    (factorize.py:452-502 restated), whose payloads are the device
    factor's bit for bit and agree with the oracle's own factorization
    (<= 1e-8 per block), and whose apply_m matches the device apply_m."""
    sp = _sp()
    a = sp.laplacian_2d(16)
    h = sp.build_hierarchy(a, 4)
    f = sp.factorize(a, h, 0.05, scheme, skip_levels=1)
    path = tmp_path / "factor.bin"
    sp.save_factor(f, path)
    g = sp.load_factor(path)
    assert (g.n, g.eps, g.scheme, g.skip_levels, g.nnz_factor) == \
        (f.n, f.eps, f.scheme, f.skip_levels, f.nnz_factor)
    assert np.array_equal(g.perm, f.perm)
    assert len(g.ops) == len(f.ops)
    for x, y in zip(f.ops, g.ops):
        assert x.kind is y.kind
        assert np.array_equal(x.dofs, y.dofs)
        for name in ("w_dofs", "lower", "panel", "q", "e_tilde"):
            if hasattr(x, name):
                assert np.array_equal(getattr(x, name), getattr(y, name)), name
    x = np.random.default_rng(6).standard_normal(f.n)
    zf, zg = f.apply_m(x), g.apply_m(x)
    # the loaded factor runs the generic scheduled apply, the engine's
    # factor the structured one: same operators, different summation order
    assert np.linalg.norm(zf - zg) <= 1e-13 * np.linalg.norm(zf)
    of, head = orc.read_spdf(path)
    assert head == {"n": f.n, "eps": f.eps, "scheme": scheme, "skip_levels": 1,
                    "n_ops": len(f.ops), "nnz_factor": f.nnz_factor}
    assert np.array_equal(of.perm, f.perm)
    kinds = {"elimination": "G", "scaling": "D", "orthogonal": "Q", "error-correction": "E"}
    for x_, y_ in zip(f.ops, of.ops):
        assert kinds[x_.kind.value] == y_.kind
        assert np.array_equal(x_.dofs, y_.dofs)
        for name in ("lower", "panel", "q", "e_tilde"):
            if hasattr(x_, name):
                assert np.array_equal(getattr(x_, name), getattr(y_, name)), name
    cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
    ref = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, 4, 0.05, scheme, 1)
    assert "".join(op.kind for op in ref.ops) == "".join(op.kind for op in of.ops)
    for x_, y_ in zip(of.ops, ref.ops):
        for name in ("lower", "panel", "e_tilde"):
            p, q = getattr(x_, name), getattr(y_, name)
            if p is not None:
                assert np.linalg.norm(p - q) <= 1e-8 * max(np.linalg.norm(q), 1e-300) + 1e-14
    zo = of.apply_m(x)
    assert np.linalg.norm(zo - zf) <= 1e-12 * np.linalg.norm(zf)
    assert np.linalg.norm(zo - ref.apply_m(x)) <= 1e-9 * np.linalg.norm(zo)


def _negate_corrections(f):
    """Flip the sign of every ErrorCorrection payload in place on the device
    (the injected mutation of test_cli.py:265-281: e_tilde -> -e_tilde)."""
    sp = _sp()
    n = 0
    for op in f.ops:
        if op.kind is not sp.OpKind.ERROR_CORRECTION:
            continue
        for v, _ in op.e_views:
            if v.rows and v.cols:
                v.buf.as_strided((v.cols, v.rows), (v.ld, 1), v.off).mul_(-1.0)
                v._host = None
                n += 1
    return n


@pytest.mark.parametrize("scheme", ["second-full", "second-superfine"])
def test_sign_flip_fault_injection_trips_quality_guard(scheme):
    """cli.py:544-556's second-order quality guard (d = 64, rho = 1,
    eps = 0.01, b = ones, tol 1e-10: n_cg <= 5) holds for the device
    factor and trips once the corrections' sign is flipped."""
    sp = _sp()
    a = sp.laplacian_2d(64)
    h = sp.build_hierarchy(a, sp.default_levels(a.n))
    b = np.ones(a.n)
    f = sp.factorize(a, h, 0.01, scheme)
    _, clean = sp.pcg(a, b, m=f.apply_m, tol=1e-10)
    assert clean.converged and clean.n_cg <= 5
    assert _negate_corrections(f) > 0
    _, bad = sp.pcg(a, b, m=f.apply_m, tol=1e-10)
    assert bad.n_cg > 5
