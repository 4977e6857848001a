"""BASELINE config C5: Q1 hexahedral elasticity with a node-blocked hierarchy.

The reference has no elasticity generator and only a scalar-dof partition
(SURVEY.md §0), so C5 is built here (``sparse.elasticity_q1``,
``partition.build_hierarchy(block=3)``) and handed to the reference's own
``factorize`` by ``tests/golden/make_golden.py c5`` (the hierarchy is an
argument of factorize.py:285).  CPU tests:

- the generator: exact symmetry, n = 3 x (free nodes), the six rigid-body
  modes are in the kernel of every row away from the clamped face;
- the node-blocked ND equals the oracle's restatement of the reference
  bisection (partition.py:135-268) run on the node graph, expanded to dofs;
- the oracle reproduces the reference's C5 golden bitwise (ranks, perm, op
  payload hashes, n_cg, residual history).

GPU: the C5 goldens run through tests/test_gpu_configs.py (config_tags), and
the rigid-body-mode near-kernel mode is checked against the oracle here.
"""

import numpy as np
import pytest

import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc
from paper_2007_00789_b200.partition import node_graph
from paper_2007_00789_b200.sparse import c5_problem, rigid_body_modes
from tests.golden_cases import hierarchy_for, load


def _sha(arr):
    import hashlib
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("ne", [6, 12])
def test_generator_rigid_body_kernel(ne):
    a, b, lv, co = c5_problem(ne)
    assert a.n == 3 * ne * (ne + 1) ** 2 == b.size
    r = rigid_body_modes(co)
    assert r.shape == (a.n, 6)
    y = a.to_scipy() @ r
    far = np.repeat(co[:, 0] > 1.5 / ne, 3)
    assert np.abs(y[far]).max() <= 1e-12 * np.abs(a.values).max()
    # clamped: the modes are NOT in the kernel next to x = 0 (SPD matrix)
    assert np.abs(y[~far]).max() > 1e-3


def test_full_c5_size():
    a, _, lv, co = c5_problem()
    assert a.n == 45000 and co.shape == (15000, 3) and lv == 9


@pytest.mark.parametrize("ne", [6, 12])
def test_node_blocked_partition_matches_oracle(ne):
    a, _, lv, _ = c5_problem(ne)
    h = sp.build_hierarchy(a, lv, block=3)
    nv, rp, ci = node_graph(a, 3)
    cl = orc.nd_hierarchy(nv, rp, ci, lv)
    assert len(cl) == len(h.clusters)
    for (cid, nodes, dep), c in zip(cl, h.clusters):
        assert cid == c.id and dep == c.depth
        assert np.array_equal((3 * np.asarray(nodes)[:, None] + np.arange(3)).ravel(), c.dofs)


def test_oracle_matches_reference_c5_golden():
    tag = "C5_ne12_L6_e0.01_second-full"
    rec, arr = load(tag)
    a = sp.sparse.c5_problem(12)[0]
    assert (a.n, a.nnz) == (rec["n"], rec["nnz_a"])
    h = hierarchy_for(tag, a, rec["levels"])
    assert _sha(np.concatenate([c.dofs for c in h.clusters]).astype(np.int64)) == \
        rec["hierarchy"]["dofs_sha"]
    cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
    f = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, rec["levels"], rec["eps"],
                      rec["scheme"], rec["skip_levels"])
    assert [lv["interfaces"] for lv in f.diagnostics["levels"]] == \
        [lv["interfaces"] for lv in rec["diagnostics"]]
    assert _sha(np.asarray(f.perm, np.int64)) == rec["perm_sha"]
    kinds = {"G": "elimination", "D": "scaling", "Q": "orthogonal", "E": "error-correction"}
    for op, want in zip(f.ops, rec["ops"]):
        assert kinds[op.kind] == want["kind"]
        for name in ("lower", "panel", "q", "e_tilde"):
            if name + "_sha" in want:
                assert _sha(getattr(op, name)) == want[name + "_sha"], name
    mv = orc.csr_matvec(a.n, a.row_ptr, a.col_idx, a.values)
    _, its, hist, *_ = orc.pcg(mv, arr["b"], f.apply_m, rec["tol"])
    assert its == rec["n_cg"] and hist == rec["residual_history"]


@pytest.mark.gpu
@pytest.mark.parametrize("ne,scheme", [(8, "second-full"), (12, "second-full"), (8, "first")])
def test_device_rigid_body_modes_match_oracle(ne, scheme):
    a, b, lv, co = c5_problem(ne)
    r = rigid_body_modes(co)
    h = sp.build_hierarchy(a, lv, block=3)
    f = sp.factorize(a, h, 0.01, scheme, skip_levels=2, near_kernel=r)
    cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
    of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, lv, 0.01, scheme, 2,
                       near_kernel=r)
    got = [[(e["cluster"], e["size_before"], e["size_after"], e["rank_f2"])
            for e in lv_["interfaces"]] for lv_ in f.diagnostics["levels"]]
    want = [[tuple(e) for e in lv_["interfaces"]] for lv_ in of.diagnostics["levels"]]
    assert got == want
    assert np.array_equal(f.perm, of.perm)
    z, zr = f.apply_m(b), of.apply_m(b)
    assert np.linalg.norm(z - zr) <= 1e-9 * np.linalg.norm(zr)
    mv = orc.csr_matvec(a.n, a.row_ptr, a.col_idx, a.values)
    _, its, *_ = orc.pcg(mv, b, of.apply_m, 1e-12)
    _, rep = sp.pcg(a, b, m=f.apply_m, tol=1e-12)
    assert abs(rep.n_cg - its) <= 1
