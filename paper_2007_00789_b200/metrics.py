"""Algorithmic work counts of one factorize + solve.

These are properties of the spaND algorithm on a given problem, not of the
implementation, so the same formula is applied to the device factor and to
the CPU oracle's factor when the two are timed side by side:

  F_elim  = sum over interiors  ns^3/3 + ns^2 nw + ns nw^2
            (Cholesky, panel TRSM, symmetric Schur/fill update)
  F_scale = sum over rescales   m^3/3 + m^2 nw
  F_rrqr  = sum over panels     sum_{k < k_stop} 4 (m-k)(nw-k) + 4 m (m-k)
  F_apply = 4 nnz_factor per apply_m (each stored entry: one multiply-add
            in the forward and one in the transposed sweep)
  F_spmv  = 2 nnz(A)
  B_apply = 16 nnz_factor + 32 n bytes per apply_m (fp64 payload read
            twice, x read/written)

``ops`` may be this package's operators (``.kind`` an ``OpKind``) or the
oracle's (``.kind`` in 'G','D','Q','E'); ``panels`` is a list of
(m, nw, k_stop) per sparsified interface in operator order.
"""

import numpy as np


def _kind(op):
    k = op.kind
    return k if isinstance(k, str) else {"elimination": "G", "scaling": "D",
                                         "orthogonal": "Q",
                                         "error-correction": "E"}[k.value]


def factor_flops(ops, panels):
    f_elim = f_scale = f_rrqr = 0.0
    panel_iter = iter(panels)
    pending_scale = []
    for op in ops:
        k = _kind(op)
        if k == "G":
            ns, nw = float(op.dofs.size), float(op.w_dofs.size)
            f_elim += ns ** 3 / 3 + ns * ns * nw + ns * nw * nw
        elif k == "D":
            pending_scale.append(float(op.dofs.size))
    for m, nw, ks in panels:
        kk = np.arange(ks, dtype=np.float64)
        f_rrqr += float(np.sum(4 * (m - kk) * np.maximum(nw - kk, 0) + 4 * m * (m - kk)))
    # rescale m^2 nw uses the same panel widths as the sparsification
    for (m, nw, _), ms in zip(panels, pending_scale):
        f_scale += ms ** 3 / 3 + ms * ms * nw
    del panel_iter
    return {"F_elim": f_elim, "F_scale": f_scale, "F_rrqr": f_rrqr,
            "F_factor": f_elim + f_scale + f_rrqr}


def solve_flops(nnz_factor, nnz_a, n_apply, n_spmv):
    return 4.0 * nnz_factor * n_apply + 2.0 * nnz_a * n_spmv


def apply_bytes(nnz_factor, n):
    return 16.0 * nnz_factor + 32.0 * n


def device_panels(factor):
    """(m, nw, k_stop) per sparsified interface of a device factor."""
    out = []
    for lv in factor.diagnostics["levels"]:
        for e in lv.get("margins", []):
            out.append((e["size_before"], e.get("n_cols", 0), e["k_stop"]))
    return out
