"""Where the device Q stores rounding residue and the oracle Q an exact zero.

    python tools/q_zero_pattern.py TAG [TAG ...]   (small fixtures)

For every orthogonal operator whose nonzero count differs from the oracle's:
shape, how many extra nonzeros, their magnitude range, and the row / column
index pattern (rows of zero panel rows? columns past k_stop?)."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tests.golden_cases import hierarchy_for, load, matrix_for  # noqa: E402


def main(tags):
    import paper_2007_00789_b200 as sp
    from oracle import spand_oracle as orc
    for tag in tags:
        rec, _ = load(tag)
        a = matrix_for(tag)
        h = hierarchy_for(tag, a, rec["levels"])
        f = sp.factorize(a, h, rec["eps"], rec["scheme"], skip_levels=rec["skip_levels"],
                         digest=False)
        cl = [(c.id, c.dofs, c.depth) for c in h.clusters]
        of = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, rec["levels"],
                           rec["eps"], rec["scheme"], rec["skip_levels"])
        shown = 0
        tot = {"ops": 0, "differ": 0, "extra": 0, "missing": 0}
        for i, (x, y) in enumerate(zip(f.ops, of.ops)):
            if x.kind.value != "orthogonal":
                continue
            tot["ops"] += 1
            q, qr = np.asarray(x.q), np.asarray(y.q)
            extra = (q != 0) & (qr == 0)
            miss = (q == 0) & (qr != 0)
            if not extra.any() and not miss.any():
                continue
            tot["differ"] += 1
            tot["extra"] += int(extra.sum())
            tot["missing"] += int(miss.sum())
            if shown < 6:
                shown += 1
                rr, cc = np.nonzero(extra)
                mags = np.abs(q[extra]) if extra.any() else np.zeros(1)
                zr = np.flatnonzero((qr != 0).sum(1) == 1)   # identity rows of the oracle Q
                zc = np.flatnonzero((qr != 0).sum(0) == 1)
                print(json.dumps({
                    "tag": tag, "op": i, "shape": list(q.shape),
                    "extra": int(extra.sum()), "missing": int(miss.sum()),
                    "mag": [float(mags.min()), float(mags.max())],
                    "rows": np.unique(rr).tolist()[:40], "cols": np.unique(cc).tolist()[:40],
                    "oracle_identity_rows": zr.tolist()[:40],
                    "oracle_identity_cols": zc.tolist()[:40],
                    "oracle_nnz": int((qr != 0).sum()), "dev_nnz": int((q != 0).sum()),
                    "oracle_rowcounts": (qr != 0).sum(1).tolist()[:64],
                    "dev_rowcounts": (q != 0).sum(1).tolist()[:64],
                }), flush=True)
        print(json.dumps({"tag": tag, "total": tot}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
