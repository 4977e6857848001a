"""Pin the CPU oracle (oracle/spand_oracle.py) to the reference's outputs.

The fixtures were frozen from the unmodified reference (spdkit 0.1.0) by
tests/golden/make_golden.py.  The oracle restates the reference with the
same NumPy/LAPACK calls, so structure, ranks and payloads must agree
bitwise (sha256); n_cg and residual histories must agree exactly.
"""

import hashlib

import numpy as np
import pytest

from oracle import spand_oracle as orc
from tests.golden_cases import load, matrix_for, small_tags


def sha(arr):
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


KIND = {"G": "elimination", "D": "scaling", "Q": "orthogonal",
        "E": "error-correction"}


@pytest.mark.parametrize("tag", small_tags())
def test_oracle_matches_reference_golden(tag):
    rec, arr = load(tag)
    a = matrix_for(tag)
    assert a.n == rec["n"] and a.nnz == rec["nnz_a"]
    cl = orc.nd_hierarchy(a.n, a.row_ptr, a.col_idx, rec["levels"])
    sizes = np.array([d.size for _, d, _ in cl], dtype=np.int64)
    depth = np.array([dep for _, _, dep in cl], dtype=np.int64)
    dofs = np.concatenate([d for _, d, _ in cl]).astype(np.int64)
    assert sha(sizes) == rec["hierarchy"]["sizes_sha"]
    assert sha(depth) == rec["hierarchy"]["depth_sha"]
    assert sha(dofs) == rec["hierarchy"]["dofs_sha"]
    f = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, rec["levels"],
                      rec["eps"], rec["scheme"], rec["skip_levels"])
    got = [[e for e in lv["interfaces"]] for lv in f.diagnostics["levels"]]
    want = [lv["interfaces"] for lv in rec["diagnostics"]]
    assert got == want
    assert sha(np.asarray(f.perm, np.int64)) == rec["perm_sha"]
    assert "".join(op.kind for op in f.ops) == rec["op_kinds"]
    assert f.nnz_factor == rec["nnz_factor"]
    for op, want in zip(f.ops, rec.get("ops", [])):
        assert KIND[op.kind] == want["kind"]
        assert sha(op.dofs) == want["dofs_sha"]
        for name in ("w_dofs", "lower", "panel", "q", "e_tilde"):
            if name + "_sha" in want:
                assert sha(getattr(op, name)) == want[name + "_sha"], name
    mv = orc.csr_matvec(a.n, a.row_ptr, a.col_idx, a.values)
    x, its, hist, done, tres, _ = orc.pcg(mv, arr["b"], f.apply_m, rec["tol"])
    assert its == rec["n_cg"]
    assert hist == rec["residual_history"]
    if "apply_m_b" in arr:
        assert np.array_equal(f.apply_m(arr["b"]), arr["apply_m_b"])


def _spdf_tags():
    import glob
    import os
    from tests.golden_cases import GOLDEN
    return sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLDEN, "*.spdf")))


@pytest.mark.parametrize("tag", _spdf_tags())
def test_oracle_spdf_reader_matches_reference_files(tag, tmp_path):
    """The checker's SPDF reader (factorize.py:452-502 restated) reads the
    reference's own files: header, perm and every payload bitwise equal to
    the sha256 the reference recorded; writing them back reproduces the
    file byte for byte (factorize.py:424-449)."""
    import os
    from tests.golden_cases import GOLDEN
    rec, _ = load(tag)
    path = os.path.join(GOLDEN, tag + ".spdf")
    f, head = orc.read_spdf(path)
    assert head["n"] == rec["n"] and head["eps"] == rec["eps"]
    assert head["scheme"] == rec["scheme"] and head["skip_levels"] == rec["skip_levels"]
    assert head["nnz_factor"] == rec["nnz_factor"] == f.nnz_factor
    assert sha(f.perm) == rec["perm_sha"]
    assert "".join(op.kind for op in f.ops) == rec["op_kinds"]
    for op, want in zip(f.ops, rec["ops"]):
        for name in ("dofs", "w_dofs", "lower", "panel", "q", "e_tilde"):
            if name + "_sha" in want:
                assert sha(getattr(op, name)) == want[name + "_sha"], name
    out = tmp_path / "back.spdf"
    orc.write_spdf(f, out, head["eps"], head["scheme"], head["skip_levels"])
    with open(path, "rb") as a, open(out, "rb") as b:
        assert a.read() == b.read()


def test_oracle_spdf_reader_rejects_corruption(tmp_path):
    import os
    from tests.golden_cases import GOLDEN
    data = open(os.path.join(GOLDEN, "lap2d_d8_L3_e0.1_k0_first.spdf"), "rb").read()
    for bad in (b"NOPE" + data[4:], data[:len(data) // 2],
                data[:4] + bytes([99]) + data[5:]):
        p = tmp_path / "bad.spdf"
        p.write_bytes(bad)
        with pytest.raises(orc.SPDFError):
            orc.read_spdf(p)
