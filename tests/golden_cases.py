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
# For every operator i and payload slot k (0 lower, 1 panel, 2 q, 3 e_tilde)
# the generator stores ||P||_F and NSK bilinear sketches u_j^T P v_j with
# seeded Rademacher u_j, v_j.  For a difference D = P_gpu - P_ref,
# E[(u^T D v)^2] = ||D||_F^2, so |sketch_gpu - sketch_ref| is an unbiased
# probe of the per-block relative Frobenius error the north star bounds
# (1e-8): NSK = 4 independent probes, compared at SK_TOL * ||P||_F.

NSK = 4
SK_TOL = 6e-8          # ~6 sigma of 1e-8 ||P||_F spread over 4 probes
SLOTS = ("lower", "panel", "q", "e_tilde")


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


# The sign of a Householder reflector (beta = -sign(x0) eta, dense.py:155-159)
# is decided on x0, which is rounding noise for a few hundred reflectors of a
# large factorization (|x0| / eta < 1e-15: mathematically zero entries); the
# CPU and the GPU can take opposite signs there.  A flipped reflector negates
# one Q column and one R row, i.e. the rest of the factorization differs by
# a diagonal sign congruence D P D' -- the same operator (apply_m agrees),
# different payload signs.  The elementwise absolute value is invariant
# under it and | |P| - |P'| | <= |P - D P' D'| elementwise, so sketches of
# |P| bound the per-block difference modulo those signs.


def op_tables(ops):
    """(fro, sketches, |P| sketches, nnz) arrays over an operator list
    (reference ops or host-materialised device ops): fro (nops, 4) with NaN
    where the slot does not exist, sketches (nops, 4, NSK), nnz (nops,)."""
    nops = len(ops)
    fro = np.full((nops, len(SLOTS)), np.nan)
    sk = np.zeros((nops, len(SLOTS), NSK))
    ska = np.zeros((nops, len(SLOTS), NSK))
    nnz = np.zeros(nops, dtype=np.int64)
    for i, op in enumerate(ops):
        for k, name in enumerate(SLOTS):
            if name in ("lower", "panel") and op.kind.value not in ("elimination", "scaling"):
                continue
            if name == "panel" and op.kind.value != "elimination":
                continue
            if name == "q" and op.kind.value != "orthogonal":
                continue
            if name == "e_tilde" and op.kind.value != "error-correction":
                continue
            p = np.asarray(getattr(op, name), dtype=np.float64)
            fro[i, k] = float(np.linalg.norm(p))
            sk[i, k] = sketch(p, i, k)
            ska[i, k] = sketch(np.abs(p), i, k)
        nnz[i] = int(op.nnz)
    return fro, sk, ska, nnz


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


def device_op_tables(ops):
    """(fro, sketches, |P| sketches) of a device factor, on the device."""
    import torch
    nops = len(ops)
    fro = np.full((nops, len(SLOTS)), np.nan)
    sk = np.zeros((nops, len(SLOTS), NSK))
    ska = np.zeros((nops, len(SLOTS), NSK))
    slot_of = {"elimination": (0, 1), "scaling": (0,), "orthogonal": (2,),
               "error-correction": (3,)}
    for i, op in enumerate(ops):
        for k in slot_of[op.kind.value]:
            p = device_payload(op, SLOTS[k])
            fro[i, k] = float(torch.linalg.norm(p)) if p.numel() else 0.0
            if p.numel():
                u, v = sketch_uv(i, k, *p.shape)
                ud = torch.as_tensor(u, device=p.device)
                vd = torch.as_tensor(v, device=p.device)
                sk[i, k] = ((ud @ p) * vd).sum(dim=1).cpu().numpy()
                ska[i, k] = ((ud @ p.abs()) * vd).sum(dim=1).cpu().numpy()
    return fro, sk, ska
