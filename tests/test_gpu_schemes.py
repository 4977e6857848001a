"""Single-block constructors of the reference API (schemes.py:199-340:
make_elimination, make_scaling, make_sparsification, local_error) on the
device kernels, against the oracle's restatement of the same steps."""

import numpy as np
import pytest

import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc


def _spd(n, rng):
    m = rng.standard_normal((n, n))
    return m @ m.T + n * np.eye(n)


@pytest.mark.gpu
def test_make_elimination_and_scaling():
    rng = np.random.default_rng(3)
    a_ss, a_ws = _spd(40, rng), rng.standard_normal((70, 40))
    op, upd = sp.make_elimination(a_ss, a_ws)
    low = orc.chol(a_ss)
    pan = np.linalg.solve(low, a_ws.T).T
    assert np.allclose(op.lower, low, rtol=1e-12, atol=1e-12)
    assert np.allclose(op.panel, pan, rtol=1e-10, atol=1e-10)
    assert np.allclose(upd, pan @ pan.T, rtol=1e-10, atol=1e-10)
    a_pp, a_pw = _spd(30, rng), rng.standard_normal((30, 90))
    sc, scaled = sp.make_scaling(a_pp, a_pw)
    z = orc.chol(a_pp)
    assert np.allclose(sc.lower, z, rtol=1e-12, atol=1e-12)
    assert np.allclose(scaled, np.linalg.solve(z, a_pw), rtol=1e-10, atol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", ["first", "second-full", "second-superfine"])
def test_make_sparsification_matches_oracle(scheme):
    rng = np.random.default_rng(11)
    w = rng.standard_normal((48, 10)) @ rng.standard_normal((10, 200))
    w += 1e-3 * rng.standard_normal((48, 200))
    res = sp.make_sparsification(w, 0.05, scheme)
    ref = orc.sparsify_panel(w, 0.05, scheme)
    assert res.rank_c == ref["rank_c"] and res.rank_f2 == ref["rank_f2"]
    assert res.n_fine == 48 - ref["rank_c"]
    assert np.allclose(np.abs(res.coarse_rows), np.abs(ref["r_coarse"]), rtol=1e-9, atol=1e-11)
    want = orc.local_error(w, ref, scheme)
    got = sp.local_error(scheme, res)
    assert abs(got - want) <= 1e-9 * max(want, 1e-300) + 1e-14
    q = res.orthogonal.q
    assert np.allclose(q.T @ q, np.eye(48), atol=1e-12)
