"""Per-operator payload comparison of the device factor against the CPU
oracle on one config (diagnostics for parity failures).

    python tools/payload_diff.py C3 [levels] [scheme] [eps]

Prints the worst operators by relative Frobenius difference; for Orthogonal
payloads also how many columns agree only up to sign (a Householder
reflector whose sign decision x0 >= 0 was taken on a rounding-level x0)."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2007_00789_b200 as sp
    from oracle import spand_oracle as orc
    name = sys.argv[1]
    a, b, lv = sp.baseline_problem(name)
    if len(sys.argv) > 2:
        lv = int(sys.argv[2])
    scheme = sys.argv[3] if len(sys.argv) > 3 else "second-full"
    eps = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-2
    h = sp.build_hierarchy(a, lv)
    f = sp.factorize(a, h, eps, scheme, digest=False)
    cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
    t0 = time.perf_counter()
    o = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, lv, eps, scheme, 4)
    print("oracle", time.perf_counter() - t0, "s", flush=True)
    rows = []
    first_bad = None
    for i, (x, y) in enumerate(zip(f.ops, o.ops)):
        for name_ in ("lower", "panel", "q", "e_tilde"):
            yv = getattr(y, name_, None)
            if yv is None or not hasattr(x, name_):
                continue
            xv = np.asarray(getattr(x, name_))
            if xv.shape != yv.shape:
                rows.append((1e9, i, x.kind.value, name_, xv.shape, "shape"))
                continue
            nrm = np.linalg.norm(yv)
            r = np.linalg.norm(xv - yv) / (nrm if nrm > 0 else 1.0)
            extra = ""
            if name_ == "q" and r > 1e-6:
                dots = np.einsum("ij,ij->j", xv, yv)
                flips = np.flatnonzero(dots < -0.5)
                extra = f"sign-flipped columns {flips[:10].tolist()} of {xv.shape[1]}"
            if r > 1e-8 and first_bad is None:
                first_bad = i
            rows.append((r, i, x.kind.value, name_, xv.shape, extra))
    rows.sort(key=lambda t: -t[0])
    for r in rows[:15]:
        print(json.dumps({"rel": r[0], "op": r[1], "kind": r[2], "payload": r[3],
                          "shape": list(r[4]), "note": r[5]}))
    print("first op above 1e-8:", first_bad, "of", len(f.ops))
    if first_bad is not None:
        y = o.ops[first_bad]
        x = f.ops[first_bad]
        print("kind", y.kind, "dofs", y.dofs.size)
        if y.kind == "Q":
            qx, qy = np.asarray(x.q), y.q
            c = np.abs(qx.T @ qy)
            diag = np.diag(c)
            bad = np.flatnonzero(np.abs(diag - 1) > 1e-8)
            print("columns off the diagonal:", bad.size, bad[:40].tolist())
            for j in bad[:12]:
                top = np.argsort(-c[j])[:3]
                print(" col", int(j), "best matches", [(int(t), float(c[j, t])) for t in top])
            # fine/coarse split of the op: n_fine = first columns
            print("sign flips (diag ~ 1 but negative dot):",
                  int(np.sum(np.einsum('ij,ij->j', qx, qy) < -0.5)))
        # diagnostics of the interfaces (margins) around that op
        ms = [e for lv_ in f.diagnostics["levels"] for e in lv_["margins"]]
        print("interfaces:", len(ms))


if __name__ == "__main__":
    main()
