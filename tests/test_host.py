"""Host-side logic on the CPU (no GPU needed).

- the C-ABI library loads and exports every symbol include/spand_b200.h
  declares (no compute calls);
- the native nested dissection (csrc/partition.cpp, reference
  partition.py:135-268) reproduces the reference's cluster lists bit for
  bit on every golden fixture, C4-L15 included;
- the native level scheduler (csrc/planner.cpp, reference factorize.py:285-366)
  produces the reference's operator order: per level the G ops of the
  interiors, then (outside skip_levels) one D per active interface and one Q
  per interface, compared with the golden op-kind strings (E ops depend on
  the ranks and are stripped);
- argument validation and SPDF parse errors raise the reference's errors
  before any device work (factorize.py:299-304, :408-467).
"""

import ctypes
import hashlib
import io
import os
import re
import struct

import numpy as np
import pytest

import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import _lib
from paper_2007_00789_b200.errors import DimensionMismatch, ParseError
from tests.golden_cases import config_tags, load, matrix_for, small_tags, hierarchy_for

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spand_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spand_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 30
    missing = [nm for nm in names if not hasattr(lib, nm)]
    assert not missing, missing
    assert lib.spand_version() > 0


def test_header_symbols_are_typed_or_handle_based():
    """Every declared entry point is either in the ctypes signature table or
    bound with explicit argtypes where it is used (handle-returning ones)."""
    handle_based = {"spand_plan_create", "spand_plan_destroy", "spand_plan_set_dofs",
                    "spand_plan_emit_begin", "spand_plan_emit_next", "spand_plan_chunk",
                    "spand_plan_pairs", "spand_plan_scatter", "spand_csr_check",
                    "spand_plan_set_group_weight", "spand_plan_set_digest",
                    "spand_mm_read", "spand_mm_csr", "spand_mm_error_span", "spand_mm_text",
                    "spand_mm_free",
                    "spand_collect_create", "spand_collect_destroy", "spand_collect_sizes",
                    "spand_collect_get", "spand_collect_apply", "spand_collect_apply_get",
                    "spand_collect_fine", "spand_collect_stats", "spand_collect_flag_sizes",
                    "spand_collect_flag_panels", "spand_collect_dataflow_sizes",
                    "spand_collect_dataflow", "spand_launch_timer_reset"}
    for nm in _declared():
        assert nm in _lib.SIGNATURES or nm in handle_based, nm


def _sha(arr):
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("tag", small_tags() + config_tags())
def test_native_hierarchy_matches_reference(tag):
    rec, _ = load(tag)
    a = matrix_for(tag)
    assert (a.n, a.nnz) == (rec["n"], rec["nnz_a"])
    h = hierarchy_for(tag, a, rec["levels"])
    sizes = np.array([c.dofs.size for c in h.clusters], dtype=np.int64)
    depth = np.array([c.depth for c in h.clusters], dtype=np.int64)
    dofs = np.concatenate([c.dofs for c in h.clusters]).astype(np.int64)
    assert [c.id for c in h.clusters] == list(range(len(h.clusters)))
    assert _sha(sizes) == rec["hierarchy"]["sizes_sha"]
    assert _sha(depth) == rec["hierarchy"]["depth_sha"]
    assert _sha(dofs) == rec["hierarchy"]["dofs_sha"]


def _plan(tag):
    from paper_2007_00789_b200.engine import NativePlan
    rec, _ = load(tag)
    a = matrix_for(tag)
    h = hierarchy_for(tag, a, rec["levels"])
    # capacity override: the RRQR group size query needs a device
    return rec, NativePlan(a, h, rec["skip_levels"], cap_override=148 * 4)


@pytest.mark.parametrize("tag", small_tags() + config_tags())
def test_scheduler_operator_order(tag):
    rec, plan = _plan(tag)
    kinds = []
    for lv in plan.level_recs:
        kinds += ["G"] * len(lv["elim"])
        if not lv["skipped"]:
            kinds += ["D"] * len(lv["active"])
            kinds += ["Q"] * len(lv["active"])
    # the leftover dense block (factorize.py:358-362) exists iff some
    # coarse dofs survive, which depends on the ranks
    if plan.nfinal and rec["final_block"] > 0:
        kinds.append("G")
    want = rec["op_kinds"].replace("E", "")
    assert "".join(kinds) == want


@pytest.mark.parametrize("tag", ["lap2d_d32_L5_e0.01_k1_second-full",
                                 "C2_L10_e0.01_second-full"])
def test_scheduler_program_is_self_consistent(tag):
    """Dry emission sizes the workspace within the a-priori bound; the real
    emission (fake base addresses, nothing launched) produces a launch list
    whose record offsets stay inside the program."""
    _, plan = _plan(tag)
    bound = plan.temp_bound
    plan.emit(1 << 40, 2 << 40, 3 << 40, 4 << 40, dry=True)
    assert 0 < plan.temp_size <= bound
    plan.emit(1 << 40, 2 << 40, 3 << 40, 4 << 40, dry=False)
    prog, lau = plan.program()
    assert lau.shape[0] == plan.n_launch > 0
    assert set(np.unique(lau[:, 0])) <= {1, 2, 3, 4, 5, 6, 12}
    for rec in lau:
        for off in rec[2:5]:
            assert 0 <= off <= prog.size
    # every level contributes at least one potrf launch (its interiors)
    assert int((lau[:, 0] == 1).sum()) >= sum(1 for lv in plan.level_recs if lv["elim"])


def test_wave_numbers_respect_id_order():
    """Sparsification waves: an interface's wave exceeds that of every
    smaller-id active neighbour (ascending-id semantics, factorize.py:209-220)."""
    _, plan = _plan("C2_L10_e0.01_second-full")
    for lv in plan.level_recs:
        if lv["skipped"]:
            continue
        wave = {p: wv for p, wv, *_ in lv["active"]}
        for p, wv, *_, nbrs in lv["active"]:
            for w in nbrs:
                if w in wave and w < p:
                    assert wave[w] < wv


def test_default_levels():
    assert sp.default_levels(16384) == 9
    assert sp.default_levels(25) == 1
    with pytest.raises(ValueError):
        sp.default_levels(1)


def test_factorize_argument_errors():
    a = sp.laplacian_2d(8)
    h = sp.build_hierarchy(a, 3)
    with pytest.raises(ValueError):
        sp.factorize(a, h, -0.1, "first")
    with pytest.raises(ValueError):
        sp.factorize(a, h, 1.5, "first")
    with pytest.raises(ValueError):
        sp.factorize(a, h, 0.1, "first", skip_levels=-1)
    with pytest.raises(ValueError):
        sp.factorize(a, h, 0.1, "third-order")
    h2 = sp.build_hierarchy(sp.laplacian_2d(9), 3)
    with pytest.raises(DimensionMismatch):
        sp.factorize(a, h2, 0.1, "first")


def _spdf_header(version=1, scheme=1, nops=0):
    return b"SPDF" + struct.pack("<HqdBHIq", version, 4, 0.1, scheme, 4, nops, 0)


@pytest.mark.parametrize("blob,msg", [
    (b"XXXX", "magic"),
    (_spdf_header(version=2), "version"),
    (_spdf_header(scheme=9), "scheme"),
    (_spdf_header()[:-3], "truncated"),
])
def test_load_factor_parse_errors(tmp_path, blob, msg):
    p = tmp_path / "bad.spdf"
    p.write_bytes(blob)
    with pytest.raises(ParseError, match=msg):
        sp.load_factor(str(p))


def test_load_factor_unknown_tag(tmp_path):
    buf = io.BytesIO()
    buf.write(_spdf_header(nops=1))
    perm = np.arange(4, dtype=np.int64)
    buf.write(struct.pack("<B", 1) + struct.pack("<q", 4) + perm.tobytes())
    buf.write(struct.pack("<B", 7))
    p = tmp_path / "tag.spdf"
    p.write_bytes(buf.getvalue())
    with pytest.raises(ParseError, match="tag"):
        sp.load_factor(str(p))


def test_matrix_market_round_trip(tmp_path):
    a = sp.laplacian_2d(6)
    p = tmp_path / "a.mtx"
    sp.write_matrix_market(str(p), a)
    b = sp.read_matrix_market(str(p))
    assert b.n == a.n
    assert np.array_equal(b.row_ptr, a.row_ptr)
    assert np.array_equal(b.col_idx, a.col_idx)
    assert np.array_equal(b.values, a.values)


def test_jacobi_prescale_unit_diagonal():
    r = np.random.default_rng(5)
    a = sp.diffusion_fv(sp.log_uniform_block_field((8, 8), 4, 3.0, r))
    b = r.standard_normal(a.n)
    s, bs = sp.jacobi_prescale(a, b)[:2]
    assert np.allclose(s.diagonal(), 1.0, rtol=0, atol=1e-15)


def test_nd_partition_rejects_bad_input():
    """The C-ABI partitioner returns -1 for a negative size (no crash)."""
    lib = _lib.load()
    z = np.zeros(4, dtype=np.int64)
    d = np.zeros(4, dtype=np.int32)
    vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = lib.spand_nd_partition(ctypes.c_int64(-1), vp(z), vp(z), 3, vp(z), vp(z), vp(d), vp(z))
    assert rc == -1


@pytest.mark.parametrize("tag", ["lap3d_d8_L6_e0.01_k1_second-full", "C5_ne12_L6_e0.01_second-full"])
def test_native_scatter_positions(tag):
    """spand_plan_scatter (the initial blocks, factorize.py:61-96) against a
    NumPy restatement: every upper-block entry of A lands at its cluster
    slots inside its block, column-major at the original block size."""
    rec, plan = _plan(tag)
    a = matrix_for(tag)
    n = a.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.row_ptr))
    cols = a.col_idx
    cl = plan.cluster_of
    slot = np.empty(n, dtype=np.int64)
    for c, dd in enumerate(plan.dofs):
        slot[dd] = np.arange(dd.size)
    ci, cj = cl[rows], cl[cols]
    up = ci <= cj
    bid = plan.bid
    want = np.full(cols.size, -1, dtype=np.int64)
    for e in np.flatnonzero(up):
        b = bid[(int(ci[e]), int(cj[e]))]
        want[e] = plan.boff[b] + slot[rows[e]] + slot[cols[e]] * plan.m0[ci[e]]
    got = np.empty(cols.size, dtype=np.int64)
    vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    lib = _lib.load()
    lib.spand_plan_scatter.argtypes = [ctypes.c_void_p] * 5
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
    cx = np.ascontiguousarray(a.col_idx, dtype=np.int64)
    cof = np.ascontiguousarray(cl, dtype=np.int64)
    assert lib.spand_plan_scatter(plan.h, vp(rp), vp(cx), vp(cof), vp(got)) == 0
    assert np.array_equal(got, want)


def test_sparse_sym_matrix_validation_errors():
    """The reference constructor's checks (sparse.py:40-58), first failing
    property reported (native pass per property)."""
    from paper_2007_00789_b200.errors import AsymmetricValues, NonpositiveDiagonal
    mk = lambda rp, ci, va: sp.SparseSymMatrix(3, np.array(rp), np.array(ci),  # noqa: E731
                                                np.array(va, dtype=float))
    good = mk([0, 2, 4, 5], [0, 1, 0, 1, 2], [2.0, -1.0, -1.0, 2.0, 1.0])
    assert good.nnz == 5
    with pytest.raises(ParseError):
        mk([0, 2, 4, 5], [0, 3, 0, 1, 2], [2.0, -1.0, -1.0, 2.0, 1.0])   # out of range
    with pytest.raises(ParseError):
        mk([0, 2, 4, 5], [1, 0, 0, 1, 2], [-1.0, 2.0, -1.0, 2.0, 1.0])   # decreasing
    with pytest.raises(AsymmetricValues):
        mk([0, 2, 4, 5], [0, 1, 0, 1, 2], [2.0, -1.0, -0.5, 2.0, 1.0])   # values
    with pytest.raises(AsymmetricValues):
        mk([0, 2, 3, 4], [0, 1, 1, 2], [2.0, -1.0, 2.0, 1.0])            # pattern
    with pytest.raises(NonpositiveDiagonal):
        mk([0, 2, 4, 5], [0, 1, 0, 1, 2], [2.0, -1.0, -1.0, 2.0, -1.0])  # sign
    with pytest.raises(NonpositiveDiagonal):                           # missing diagonal
        sp.SparseSymMatrix(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))


@pytest.mark.parametrize("shape,block,seed", [((24, 24, 24), 8, 3), ((16, 16), 4, 2)])
def test_oracle_generator_matches_package(shape, block, seed):
    """bench.py's CPU legs build their sample with the oracle's generator
    (they must not load the product); it is the package's construction bit
    for bit."""
    from oracle import spand_oracle as orc
    from paper_2007_00789_b200 import sparse as S
    n, rp, ci, va, b = orc.fv_block_field_problem(shape, block, 3.0, seed)
    rng = np.random.default_rng(seed)
    a = S.diffusion_fv(S.log_uniform_block_field(shape, block, 3.0, rng))
    assert a.n == n
    assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
    assert np.array_equal(a.values, va)
    assert np.array_equal(rng.standard_normal(n), b)


def test_oversized_interface_raises_before_launch():
    """An interface taller than the device RRQR's limit (rrqr.cu kMaxM) is
    rejected with a typed error before any allocation or launch (so it runs
    without a GPU); the reference (dense.py:117) has no cap."""
    from paper_2007_00789_b200.engine import MAX_PANEL_ROWS
    from paper_2007_00789_b200.partition import Cluster, PartitionHierarchy
    big = MAX_PANEL_ROWS + 10
    n = big + 2
    a = sp.from_coo(n, np.arange(n), np.arange(n), np.full(n, 2.0))
    cl = [Cluster(id=0, dofs=np.arange(2, n), depth=0),
          Cluster(id=1, dofs=np.array([0]), depth=1),
          Cluster(id=2, dofs=np.array([1]), depth=1)]
    h = PartitionHierarchy(1, n, cl, np.zeros(n + 1, np.int64), np.zeros(0, np.int64))
    with pytest.raises(sp.PanelTooLarge) as exc:
        sp.factorize(a, h, 0.01, "first", skip_levels=0)
    assert exc.value.rows == big and exc.value.cluster == 0
    assert isinstance(exc.value, NotImplementedError)


def test_one_sided_explicit_zero_is_accepted():
    """The reference's symmetry test compares VALUES ((csr != csr.T).nnz,
    sparse.py:52-53): a stored zero whose mirror is absent equals the
    implicit zero and is accepted; a one-sided nonzero is rejected.  The
    native hierarchy of such a pattern equals the oracle's."""
    from oracle import spand_oracle as orc
    a = sp.laplacian_2d(6)
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    r = np.concatenate([rows, [0]])
    c = np.concatenate([a.col_idx, [20]])
    v = np.concatenate([a.values, [0.0]])
    z = sp.from_coo(a.n, r, c, v)
    assert z.nnz == a.nnz + 1
    with pytest.raises(sp.AsymmetricValues):
        sp.from_coo(a.n, r, c, np.concatenate([a.values, [1e-3]]))
    h = sp.build_hierarchy(z, 3)
    cl = orc.nd_hierarchy(z.n, z.row_ptr, z.col_idx, 3)
    assert [c_.dofs.tolist() for c_ in h.clusters] == [d.tolist() for _, d, _ in cl]
    assert [c_.depth for c_ in h.clusters] == [dep for _, _, dep in cl]


_MM_CASES = {
    "ok": "%%MatrixMarket matrix coordinate real symmetric\n% c\n\n3 3 4\n1 1 4.0\n2 1 -1\n"
          "2 2 4e0\n3 3 1_0.5\n",
    "ok_mirror": "%%MatrixMarket matrix coordinate real symmetric\n2 2 4\n1 1 2\n2 1 -.5\n"
                 "1 2 -0.5\n2 2 3\n",
    "ok_crlf": "%%MatrixMarket Matrix Coordinate REAL Symmetric\r\n2 2 3\r\n1 1 2\r\n"
               "2 1 1e-3\r\n2 2 +3.\r\n",
    "bad_header": "%%MatrixMarkt matrix coordinate real symmetric\n1 1 1\n1 1 1\n",
    "bad_format": "%%MatrixMarket matrix array real symmetric\n1 1 1\n1 1 1\n",
    "general": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n",
    "bad_size": "%%MatrixMarket matrix coordinate real symmetric\n2 2\n1 1 1\n",
    "empty_size": "%%MatrixMarket matrix coordinate real symmetric\n% only comments\n",
    "rect": "%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n",
    "short": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1\n2 2 1\n",
    "bad_line": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n2 2\n",
    "bad_number": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n2 2 0x1p3\n",
    "comment_in_entries": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n"
                          "% no\n",
    "range": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n3 1 1\n",
    "dup": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1\n2 2 1\n1 1 2\n",
    "asym": "%%MatrixMarket matrix coordinate real symmetric\n2 2 4\n1 1 1\n1 2 0.25\n"
            "2 2 1\n2 1 0.5\n",
    "first_error_wins": "%%MatrixMarket matrix coordinate real symmetric\n2 2 4\n1 1 1\n"
                        "1 2 1\n2 1 2\n2 2 x\n",
    "inf_nan": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 inf\n2 2 NaN\n",
}


@pytest.mark.parametrize("case", sorted(_MM_CASES))
def test_matrix_market_reader_matches_reference_semantics(tmp_path, case):
    """The native reader (csrc/mmio.cpp) against the oracle's restatement of
    the reference reader (sparse.py:98-160): the same CSR, or the same error
    class and message, for valid files, CRLF, comments, number syntax
    (Python int()/float()), every error kind, and first-error-wins order."""
    from oracle import spand_oracle as orc
    from paper_2007_00789_b200 import errors as E
    p = tmp_path / f"{case}.mtx"
    p.write_bytes(_MM_CASES[case].encode())
    try:
        want = orc.mm_read(str(p))
        werr = None
    except orc.MMError as exc:
        want, werr = None, exc
    if werr is not None:
        with pytest.raises(getattr(E, werr.kind)) as got:
            sp.read_matrix_market(str(p))
        assert str(got.value) == str(werr)
        return
    try:
        a = sp.read_matrix_market(str(p))
    except (E.NonpositiveDiagonal, E.AsymmetricValues) as exc:
        # the file parses; the SparseSymMatrix constructor's checks then
        # apply to both readers' output alike
        with pytest.raises(type(exc)):
            sp.SparseSymMatrix(*want)
        return
    n, rp, ci, va = want
    assert a.n == n and np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci)
    assert np.array_equal(a.values, va, equal_nan=True)


def test_matrix_market_reader_large_file(tmp_path):
    """C2 written and read back: identical CSR (the multi-threaded path)."""
    a = sp.laplacian_3d(32)
    p = tmp_path / "c2.mtx"
    sp.write_matrix_market(str(p), a)
    b = sp.read_matrix_market(str(p))
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)
