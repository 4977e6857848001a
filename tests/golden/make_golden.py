"""Freeze golden vectors from the UNMODIFIED reference (spdkit 0.1.0).

Test infrastructure only.  Runs in the build container, where the reference
is importable from /root/reference/pkg/src (it does not exist on the GPU
box, so its outputs travel as the fixtures written here):

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py small
    ... python tests/golden/make_golden.py config C2 second-full 1e-2 [levels]
    ... python tests/golden/make_golden.py c5 12|24

Inputs come from this package's generators (``baseline_problem``;
``laplacian_2d`` is bit-identical to the reference's) and are handed to the
reference's own ``build_hierarchy``/``factorize``/``pcg``.  Everything is
seeded (``np.random.default_rng``), so fixtures are reproducible; the
numpy/scipy versions used are recorded in each file.

Per run we store: cluster structure (full arrays for small cases, sizes +
sha256 for the big ones), per-level diagnostics (interface ranks, rank_f2),
the factor's perm, per-op payload sha256 and Frobenius norms, nnz_factor,
n_cg, the residual history and timings (1 BLAS thread, this container).
Every run also stores, per operator, the Frobenius norms and four
bilinear sketches of the payloads' invariant forms and nnz of each payload
(``op_fro5``/``op_ska5``/``op_nnz`` in the .npz, see tests/golden_cases.py),
apply_m(b) and the PCG solution x, so the full-size configs are checked
per block without storing their factors.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import spdkit  # noqa: E402  (the reference, via PYTHONPATH)
from spdkit.schemes import OpKind  # noqa: E402

from paper_2007_00789_b200 import sparse as gen  # noqa: E402
from tests.golden_cases import op_tables, rank_c_of  # noqa: E402


def sha(arr):
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256()
    h.update(str(arr.dtype).encode())
    h.update(str(arr.shape).encode())
    h.update(arr.tobytes())
    return h.hexdigest()


def to_ref(a):
    return spdkit.SparseSymMatrix(a.n, a.row_ptr.copy(), a.col_idx.copy(),
                                  a.values.copy())


def hierarchy_record(h, full):
    sizes = np.array([c.dofs.size for c in h.clusters], dtype=np.int64)
    depth = np.array([c.depth for c in h.clusters], dtype=np.int64)
    dofs = (np.concatenate([c.dofs for c in h.clusters]).astype(np.int64)
            if h.clusters else np.empty(0, np.int64))
    rec = {"levels": int(h.levels), "n": int(h.n),
           "n_clusters": len(h.clusters),
           "sizes_sha": sha(sizes), "depth_sha": sha(depth),
           "dofs_sha": sha(dofs)}
    arrays = {"cl_sizes": sizes, "cl_depth": depth, "cl_dofs": dofs}
    return rec, (arrays if full else {"cl_sizes": sizes, "cl_depth": depth})


def op_record(op):
    rec = {"kind": op.kind.value, "dofs_sha": sha(op.dofs)}
    for name in ("w_dofs", "lower", "panel", "q", "e_tilde"):
        if hasattr(op, name):
            v = getattr(op, name)
            rec[name + "_sha"] = sha(v)
            rec[name + "_shape"] = list(np.shape(v))
            if name != "w_dofs" and name != "dofs":
                rec[name + "_fro"] = float(np.linalg.norm(v))
    rec["nnz"] = int(op.nnz)
    return rec


def to_ref_hierarchy(h):
    """Our (node-blocked) hierarchy as the reference's own PartitionHierarchy
    object: ``factorize`` takes the hierarchy as an argument
    (factorize.py:285), so both sides see the same clusters."""
    from spdkit.partition import Cluster as RCluster, PartitionHierarchy as RPH
    cl = [RCluster(id=c.id, dofs=np.asarray(c.dofs, dtype=np.int64), depth=c.depth)
          for c in h.clusters]
    return RPH(h.levels, h.n, cl, h._adj_ptr, h._adj_idx)


def run_case(tag, a, b, levels, eps, scheme, skip_levels=4, tol=1e-12,
             full=True, store_factor=False, store_ops=True, hierarchy=None,
             sketches=True):
    ra = to_ref(a)
    t0 = time.perf_counter()
    h = (spdkit.build_hierarchy(ra, levels) if hierarchy is None
         else to_ref_hierarchy(hierarchy))
    t_hier = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = spdkit.factorize(ra, h, eps, scheme, skip_levels=skip_levels)
    t_fact = time.perf_counter() - t0
    x, rep = spdkit.pcg(ra, b, m=f.apply_m, tol=tol)
    t_apply = None
    if a.n <= 300000:
        t0 = time.perf_counter()
        z = f.apply_m(b)
        t_apply = time.perf_counter() - t0
    else:
        z = None
    hrec, harr = hierarchy_record(h, full)
    rec = {
        "tag": tag, "n": int(a.n), "nnz_a": int(a.nnz), "levels": int(levels),
        "eps": float(eps), "scheme": scheme, "skip_levels": int(skip_levels),
        "tol": tol, "hierarchy": hrec,
        "diagnostics": [
            {"level": lv["level"], "interior_clusters": lv["interior_clusters"],
             "interior_dofs": lv["interior_dofs"], "skipped": lv["skipped"],
             "interfaces": [[e["cluster"], e["size_before"], e["size_after"],
                             e["rank_f2"]] for e in lv["interfaces"]]}
            for lv in f.diagnostics["levels"]],
        "final_block": f.diagnostics["final_block"],
        "perm_sha": sha(np.asarray(f.perm, dtype=np.int64)),
        "n_ops": len(f.ops),
        "op_kinds": "".join("GDQE"[["elimination", "scaling", "orthogonal",
                                    "error-correction"].index(op.kind.value)]
                            for op in f.ops),
        "nnz_factor": int(f.nnz_factor),
        "mu": float(spdkit.memory_ratio(f, ra)),
        "n_cg": int(rep.n_cg), "converged": bool(rep.converged),
        "residual_history": [float(v) for v in rep.residual_history],
        "true_residual": float(rep.true_residual),
        "t_hier_s": t_hier, "t_factor_s": t_fact,
        "t_solve_s": float(rep.solve_seconds), "t_apply_m_s": t_apply,
        "versions": {"numpy": np.__version__, "scipy": scipy.__version__,
                     "spdkit": spdkit.__version__},
        "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
    }
    if store_ops:
        rec["ops"] = [op_record(op) for op in f.ops]
    arrays = dict(harr)
    if sketches:
        # per-operator ||P||_F, bilinear sketches and nnz of every payload
        # (tests/golden_cases.py:op_tables): full-size per-block parity
        fro, ska, nnz = op_tables(f.ops, rank_c_of(f.diagnostics["levels"]))
        arrays["op_fro5"], arrays["op_ska5"], arrays["op_nnz"] = fro, ska, nnz
        rec["digests"] = [lv["digest"] for lv in f.diagnostics["levels"]]
    arrays["perm"] = np.asarray(f.perm, dtype=np.int32 if a.n < 2**31 else np.int64)
    arrays["b"] = np.asarray(b)
    if z is not None:
        arrays["apply_m_b"] = z
    arrays["x"] = x
    base = os.path.join(HERE, tag)
    with open(base + ".json", "w") as fh:
        json.dump(rec, fh, indent=1)
    np.savez_compressed(base + ".npz", **arrays)
    if store_factor:
        spdkit.save_factor(f, base + ".spdf")
    print(json.dumps({k: rec[k] for k in ("tag", "n", "n_cg", "mu",
                                          "t_hier_s", "t_factor_s",
                                          "t_solve_s")}), flush=True)
    return rec


def small():
    schemes = ["first", "second-full", "second-superfine"]
    rng = np.random.default_rng(11)
    # tiny cases: full factor files for the load/apply path
    for d, lv, eps, skip in [(8, 3, 0.1, 0), (16, 4, 0.05, 1),
                             (16, 4, 0.0, 0), (32, 5, 0.01, 1)]:
        a = gen.laplacian_2d(d)
        b = rng.standard_normal(a.n)
        for s in schemes:
            run_case(f"lap2d_d{d}_L{lv}_e{eps:g}_k{skip}_{s}", a, b, lv, eps,
                     s, skip_levels=skip, store_factor=True)
    # 3D and high-contrast small cases (same generators as C2-C4)
    a = gen.laplacian_3d(8)
    b = rng.standard_normal(a.n)
    for s in schemes:
        run_case(f"lap3d_d8_L6_e0.01_k1_{s}", a, b, 6, 0.01, s, skip_levels=1,
                 store_factor=True)
    r2 = np.random.default_rng(2)
    a = gen.diffusion_fv(gen.log_uniform_block_field((64, 64), 8, 3.0, r2))
    b = r2.standard_normal(a.n)
    run_case("hc2d_d64_L8_e0.01_k4_second-full", a, b, 8, 0.01, "second-full")
    r3 = np.random.default_rng(3)
    a = gen.diffusion_fv(gen.log_uniform_block_field((16, 16, 16), 4, 3.0, r3))
    b = r3.standard_normal(a.n)
    run_case("hc3d_d16_L8_e0.01_k2_second-full", a, b, 8, 0.01, "second-full",
             skip_levels=2)
    # C1 (BASELINE config 0), all three schemes
    a, b, lv = gen.baseline_problem("C1")
    for s in schemes:
        run_case(f"C1_{s}", a, b, lv, 0.01, s)


def config(name, scheme, eps, levels=None):
    a, b, lv = gen.baseline_problem(name)
    if levels is not None:
        lv = int(levels)
    run_case(f"{name}_L{lv}_e{eps:g}_{scheme}", a, b, lv, float(eps), scheme,
             full=(a.n <= 40000), store_ops=(a.n <= 40000))


def c5(ne):
    """BASELINE config C5 (Q1 elasticity, node-blocked hierarchy built by
    this package's native ND on the node graph, handed to the reference)."""
    from paper_2007_00789_b200.partition import build_hierarchy
    a, b, lv, _ = gen.c5_problem(ne)
    h = build_hierarchy(a, lv, block=3)
    tag = f"C5_ne{ne}_L{lv}_e0.01_second-full"
    run_case(tag, a, b, lv, 0.01, "second-full", full=(a.n <= 40000),
             store_ops=(a.n <= 40000), hierarchy=h)


def local_errors():
    """Per-interface local errors (collect_local_errors=True,
    factorize.py:338-339) of small cases, all schemes."""
    out = {}
    for d, lv, eps, skip in [(16, 4, 0.1, 0), (32, 5, 0.05, 1)]:
        a = gen.laplacian_2d(d)
        ra = to_ref(a)
        h = spdkit.build_hierarchy(ra, lv)
        for s in ["first", "second-full", "second-superfine"]:
            f = spdkit.factorize(ra, h, eps, s, skip_levels=skip, collect_local_errors=True)
            out[f"lap2d_d{d}_L{lv}_e{eps:g}_k{skip}_{s}"] = [
                [e["cluster"], e["local_error"]] for lvd in f.diagnostics["levels"]
                for e in lvd["interfaces"]]
    with open(os.path.join(HERE, "local_errors.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    if sys.argv[1] == "small":
        small()
    elif sys.argv[1] == "local_errors":
        local_errors()
    elif sys.argv[1] == "c5":
        c5(int(sys.argv[2]))
    else:
        config(sys.argv[2], sys.argv[3], float(sys.argv[4]),
               sys.argv[5] if len(sys.argv) > 5 else None)
