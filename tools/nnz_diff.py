"""Per-operator nnz of the device factor against the reference goldens.

    python tools/nnz_diff.py TAG [TAG ...]

Prints, per operator kind and payload, how many operators differ and the
summed difference, plus the first few differing operators with their
per-payload counts (device views) -- to locate where the device factor
stores rounding noise where the reference has exact zeros."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tests.golden_cases import hierarchy_for, load, matrix_for  # noqa: E402


def main(tags):
    import paper_2007_00789_b200 as sp
    out = {}
    for tag in tags:
        rec, arr = load(tag)
        if "op_nnz" in arr:
            want = arr["op_nnz"]
        elif "ops" in rec:
            want = np.array([o["nnz"] for o in rec["ops"]])
        else:
            print(tag, "no per-op nnz in the golden")
            continue
        a = matrix_for(tag)
        h = hierarchy_for(tag, a, rec["levels"])
        f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"],
                         digest=False)
        got = np.array([op.nnz for op in f.ops])
        kinds = np.array([op.kind.value for op in f.ops])
        d = got - want
        summ = {}
        for k in np.unique(kinds):
            sel = kinds == k
            summ[k] = {"ops": int(sel.sum()), "differ": int((d[sel] != 0).sum()),
                       "sum_diff": int(d[sel].sum()), "abs_diff": int(np.abs(d[sel]).sum())}
        ex = []
        for i in np.flatnonzero(d)[:8]:
            op = f.ops[int(i)]
            row = {"i": int(i), "kind": op.kind.value, "got": int(got[i]), "want": int(want[i])}
            for name in ("lower", "panel", "q", "e_tilde"):
                if hasattr(op, name):
                    p = np.asarray(getattr(op, name))
                    row[name] = [int(np.count_nonzero(p)), list(p.shape),
                                 float(np.min(np.abs(p[p != 0]))) if np.any(p) else 0.0]
            ex.append(row)
        out[tag] = {"nnz": int(got.sum()), "ref": int(want.sum()), "by_kind": summ,
                    "examples": ex}
        print(json.dumps({tag: out[tag]}), flush=True)
    return out


if __name__ == "__main__":
    main(sys.argv[1:])
