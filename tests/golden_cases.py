"""Rebuild the inputs of the fixtures frozen by tests/golden/make_golden.py."""

import glob
import json
import os

import numpy as np

from paper_2007_00789_b200 import sparse as gen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(tag):
    with open(os.path.join(GOLDEN, tag + ".json")) as fh:
        rec = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, tag + ".npz")))
    return rec, arrays


def matrix_for(tag):
    """Same construction make_golden.py used for ``tag``."""
    if tag.startswith("lap2d_d"):
        d = int(tag.split("_")[1][1:])
        return gen.laplacian_2d(d)
    if tag.startswith("lap3d_d"):
        d = int(tag.split("_")[1][1:])
        return gen.laplacian_3d(d)
    if tag.startswith("hc2d_d64"):
        r = np.random.default_rng(2)
        return gen.diffusion_fv(gen.log_uniform_block_field((64, 64), 8, 3.0, r))
    if tag.startswith("hc3d_d16"):
        r = np.random.default_rng(3)
        return gen.diffusion_fv(
            gen.log_uniform_block_field((16, 16, 16), 4, 3.0, r))
    if tag.startswith("C5_ne"):
        return gen.c5_problem(int(tag.split("_")[1][2:]))[0]
    name = tag.split("_")[0]
    return gen.baseline_problem(name)[0]


def hierarchy_for(tag, a, levels):
    """The hierarchy make_golden.py handed to the reference: node-blocked
    (3 dofs per node) for the C5 elasticity cases, plain ND otherwise."""
    from paper_2007_00789_b200.partition import build_hierarchy
    return build_hierarchy(a, levels, block=3 if tag.startswith("C5") else 1)


def small_tags():
    tags = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        tag = os.path.basename(p)[:-5]
        if tag.startswith(("lap2d", "lap3d", "hc2d", "hc3d", "C1_")):
            tags.append(tag)
    return tags


def config_tags():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "C[2-5]_*.json"))):
        out.append(os.path.basename(p)[:-5])
    return out


# --------------------------------------------------------------------------
# Per-operator payload sketches (full-size parity without storing factors).
#
# Two rounding-level decisions make a correct factorization differ from the
# reference's by more than rounding, without changing the operator:
#
# * the sign of a Householder reflector (beta = -sign(x0) eta,
#   dense.py:155-159) is decided on x0, which is rounding noise for a few
#   hundred reflectors of a large factorization (|x0| / eta < 1e-15); the two
#   choices are different reflections.  The factored part is unique up to
#   signs (R rows < k_stop, Q's factored columns), so downstream blocks differ
#   by diagonal sign congruences D P D';
# * the unfactored columns of Q (the fine complement, reflector positions
#   >= k_stop) are only ONE orthonormal basis of the complement of the
#   factored columns, and the rows of e_tilde = Q_f^T W live in that basis:
#   a flipped reflector rotates both.
#
# The sketched quantities are therefore invariant forms, each equal to the
# payload up to those transformations:
#   0 |L|       (elimination / scaling lower)     sign congruence
#   1 |panel|   (elimination panel)               sign congruence
#   2 |Q_c|     (coarse = factored columns of q)  signs
#   3 |Q_f Q_f^T| (projector on the fine space)   sign congruence, basis-free
#   4 |Q_f[:, :r] E| (correction mapped back)     sign congruence, basis-free
# For each, ||X||_F and NSK bilinear sketches u^T |X| v with seeded
# Rademacher u, v: for a difference D, E[(u^T D v)^2] = ||D||_F^2 and
# | |X| - |Y| | <= |X - Y| elementwise, so the sketch difference probes the
# per-block relative Frobenius error the north star bounds (1e-8).

NSK = 4
SK_TOL = 6e-8          # ~6 sigma of 1e-8 ||X||_F spread over 4 probes
SLOTS = ("lower", "panel", "q_coarse", "q_fine_projector", "correction")


def sketch_uv(i, k, r, c):
    rng = np.random.default_rng([int(i), int(k)])
    u = (rng.integers(0, 2, size=(NSK, r)) * 2 - 1).astype(np.float64)
    v = (rng.integers(0, 2, size=(NSK, c)) * 2 - 1).astype(np.float64)
    return u, v


def sketch(p, i, k):
    """NSK bilinear probes of the (host) matrix ``p`` for operator i, slot k."""
    p = np.asarray(p, dtype=np.float64)
    if p.ndim != 2 or p.size == 0:
        return np.zeros(NSK)
    u, v = sketch_uv(i, k, *p.shape)
    return np.einsum("jc,jc->j", u @ p, v)


def _kind(op):
    k = op.kind
    return k if isinstance(k, str) else {"elimination": "G", "scaling": "D",
                                         "orthogonal": "Q", "error-correction": "E"}[k.value]


def invariant_forms(ops, rank_c, xp=np):
    """Yield (op index, slot, matrix) of the invariant forms above.
    ``rank_c``: per Orthogonal op (operator order), its coarse count
    (diagnostics size_after).  ``xp``: numpy, or a converter of device
    payloads (see device_op_tables)."""
    qi = 0
    last_qf = None
    for i, op in enumerate(ops):
        k = _kind(op)
        if k in ("G", "D"):
            yield i, 0, xp["lower"](op)
            if k == "G":
                yield i, 1, xp["panel"](op)
        elif k == "Q":
            q = xp["q"](op)
            kc = int(rank_c[qi])
            qi += 1
            nf = q.shape[0] - kc
            yield i, 2, q[:, nf:]
            qf = q[:, :nf]
            yield i, 3, qf @ qf.T
            last_qf = qf
        else:
            e = xp["e_tilde"](op)
            yield i, 4, last_qf[:, :e.shape[0]] @ e


def _np_access():
    return {"lower": lambda op: np.asarray(op.lower, dtype=np.float64),
            "panel": lambda op: np.asarray(op.panel, dtype=np.float64),
            "q": lambda op: np.asarray(op.q, dtype=np.float64),
            "e_tilde": lambda op: np.asarray(op.e_tilde, dtype=np.float64)}


def op_tables(ops, rank_c):
    """(fro, |X| sketches, nnz) over an operator list (reference ops, or
    host-materialised device ops): fro (nops, 5) with NaN where the slot
    does not exist, sketches (nops, 5, NSK), nnz (nops,)."""
    nops = len(ops)
    fro = np.full((nops, len(SLOTS)), np.nan)
    ska = np.zeros((nops, len(SLOTS), NSK))
    for i, k, x in invariant_forms(ops, rank_c, _np_access()):
        ax = np.abs(x)
        fro[i, k] = float(np.linalg.norm(x))
        ska[i, k] = sketch(ax, i, k)
    nnz = np.array([int(op.nnz) for op in ops], dtype=np.int64)
    return fro, ska, nnz


def rank_c_of(diagnostics_levels):
    """Coarse counts of the sparsified interfaces, in operator order."""
    return [e["size_after"] if isinstance(e, dict) else e[2]
            for lv in diagnostics_levels for e in lv["interfaces"]]


def device_payload(op, name):
    """The logical payload matrix of a device operator as a CUDA tensor
    (no host copy): MatView windows (column-major, optionally rotated and
    transposed), panels stacked by rows, corrections by columns."""
    import torch
    from paper_2007_00789_b200.schemes import MatView

    def mat(v):
        if not isinstance(v, MatView):
            return torch.as_tensor(np.asarray(v, dtype=np.float64), device="cuda")
        if v.rows == 0 or v.cols == 0:
            m = torch.zeros((v.rows, v.cols), dtype=torch.float64, device=v.buf.device)
        else:
            m = v.buf.as_strided((v.rows, v.cols), (1, v.ld), v.off)
        if v.rot:
            m = torch.cat([m[:, v.rot:], m[:, :v.rot]], dim=1)
        return m.t() if v.trans else m

    if name == "panel":
        views = op.panel_views if op._panel is not None else None
        if views is None:
            return mat(op.panel)
        if not views:
            return torch.zeros((op.w_dofs.size, op.dofs.size), dtype=torch.float64,
                               device="cuda")
        return torch.cat([mat(v) for v, _ in views], dim=0)
    if name == "e_tilde":
        views = op.e_views if op._e is not None else None
        if views is None:
            return mat(op.e_tilde)
        return torch.cat([mat(v) for v, _ in views], dim=1)
    if name == "lower":
        return mat(op._lower)
    return mat(op._q)


def device_op_tables(ops, rank_c):
    """op_tables() of a device factor (fro, |X| sketches), on the device."""
    import torch
    nops = len(ops)
    fro = np.full((nops, len(SLOTS)), np.nan)
    ska = np.zeros((nops, len(SLOTS), NSK))
    acc = {name: (lambda op, nm=name: device_payload(op, nm))
           for name in ("lower", "panel", "q", "e_tilde")}
    for i, k, x in invariant_forms(ops, rank_c, acc):
        fro[i, k] = float(torch.linalg.norm(x)) if x.numel() else 0.0
        if x.numel():
            u, v = sketch_uv(i, k, *x.shape)
            ud = torch.as_tensor(u, device=x.device)
            vd = torch.as_tensor(v, device=x.device)
            ska[i, k] = ((ud @ x.abs()) * vd).sum(dim=1).cpu().numpy()
    return fro, ska
