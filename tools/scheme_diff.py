"""First operator at which two schemes' factors differ bitwise (excluding
the corrections), with per-kind counts -- the trailing matrix is the same
for every scheme (test_factorize.py:104-137), so only E ops may differ.

    python tools/scheme_diff.py [d] [eps] [schemeA] [schemeB]"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2007_00789_b200 as sp
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    sa = sys.argv[3] if len(sys.argv) > 3 else "first"
    sb = sys.argv[4] if len(sys.argv) > 4 else "second-superfine"
    a = sp.laplacian_2d(d)
    h = sp.build_hierarchy(a, sp.default_levels(a.n))
    fa = sp.factorize(a, h, eps, sa)
    fb = sp.factorize(a, h, eps, sb)
    ob = [op for op in fb.ops if op.kind is not sp.OpKind.ERROR_CORRECTION]
    oa = [op for op in fa.ops if op.kind is not sp.OpKind.ERROR_CORRECTION]
    print("ops", len(oa), len(ob))
    qi = 0
    shown = 0
    for i, (x, y) in enumerate(zip(oa, ob)):
        for name in ("lower", "panel", "q"):
            if not hasattr(x, name):
                continue
            px, py = np.asarray(getattr(x, name)), np.asarray(getattr(y, name))
            if px.shape != py.shape:
                print(i, x.kind.value, name, "shape", px.shape, py.shape)
                shown += 1
                continue
            if not np.array_equal(px, py):
                diff = np.argwhere(px != py)
                rel = np.linalg.norm(px - py) / max(np.linalg.norm(py), 1e-300)
                print(i, x.kind.value, name, px.shape, "entries differ", diff.shape[0],
                      "first", diff[:3].tolist(), "rel", rel)
                if name == "q":
                    cols = np.unique(diff[:, 1])
                    print("   q columns differing", cols[:20].tolist(), "of", px.shape[1])
                shown += 1
        if shown > 12:
            break
    print("digests", [lv["digest"][:8] for lv in fa.diagnostics["levels"]])
    print("digests", [lv["digest"][:8] for lv in fb.diagnostics["levels"]])
    for lv in fb.diagnostics["levels"]:
        print(lv["level"], [(e["cluster"], e["size_before"], e["size_after"], e["rank_f2"])
                            for e in lv["interfaces"]][:6])


if __name__ == "__main__":
    main()
