"""Block operators of the factor (reference `schemes.py:48-196`).

Same classes, kinds and attributes as the reference (``dofs``, ``w_dofs``,
``lower``, ``panel``, ``q``, ``e_tilde``, ``nnz``, ``apply_inv``,
``apply_inv_t``), but the payloads live on the B200: each attribute is a
``MatView`` (a window into a device buffer, column-major, possibly
transposed) materialised to NumPy only when a caller asks for it.  The
preconditioner never touches the host copies; it runs the batched apply
plan of ``apply.py`` on the device.
"""

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .dense import SchemeKind

__all__ = ["SchemeKind", "OpKind", "MatView", "BlockOperator", "Elimination",
           "Scaling", "Orthogonal", "ErrorCorrection"]


class OpKind(Enum):
    ELIMINATION = "elimination"
    SCALING = "scaling"
    ORTHOGONAL = "orthogonal"
    ERROR_CORRECTION = "error-correction"


class MatView:
    """Logical matrix stored column-major in a device buffer.

    ``buf`` is a 1-D fp64 device tensor; the stored matrix has ``rows`` x
    ``cols`` entries at ``buf[off + i + j * ld]``.  The logical matrix is the
    stored one with its columns rotated left by ``rot`` (column j is stored
    column (j + rot) % cols) and then transposed when ``trans``.
    """

    __slots__ = ("buf", "off", "ld", "rows", "cols", "trans", "rot", "_host")

    def __init__(self, buf, off, ld, rows, cols, trans=False, rot=0):
        self.buf, self.off, self.ld = buf, int(off), int(ld)
        self.rows, self.cols = int(rows), int(cols)
        self.trans, self.rot = bool(trans), int(rot)
        self._host = None

    @property
    def shape(self):
        return (self.cols, self.rows) if self.trans else (self.rows, self.cols)

    @property
    def addr(self):
        return self.buf.data_ptr() + 8 * self.off

    def host(self):
        if self._host is None:
            if self.rows == 0 or self.cols == 0:
                m = np.zeros((self.rows, self.cols))
            else:
                span = (self.cols - 1) * self.ld + self.rows
                flat = self.buf[self.off:self.off + span].cpu().numpy()
                m = np.lib.stride_tricks.as_strided(
                    flat, shape=(self.rows, self.cols),
                    strides=(8, 8 * self.ld)).copy()
            if self.rot:
                m = np.concatenate([m[:, self.rot:], m[:, :self.rot]], axis=1)
            self._host = np.ascontiguousarray(m.T if self.trans else m)
        return self._host

    def count_nonzero(self):
        """Nonzeros of the stored window, counted on the device."""
        if self.rows == 0 or self.cols == 0:
            return 0
        if self._host is not None:
            return int(np.count_nonzero(self._host))
        span = (self.cols - 1) * self.ld + self.rows
        flat = self.buf[self.off:self.off + span]
        win = flat.as_strided((self.cols, self.rows), (self.ld, 1))
        return int((win != 0).sum().item())


def host_view(arr):
    """MatView over a host ndarray uploaded on demand (loaded factors)."""
    return arr


def _as_host(x):
    return x.host() if isinstance(x, MatView) else x


class BlockOperator:
    """One factor of the inverse lower-triangular product."""

    kind = None

    def apply_inv(self, x):
        from .apply import apply_single
        apply_single(self, x, transpose=False)

    def apply_inv_t(self, x):
        from .apply import apply_single
        apply_single(self, x, transpose=True)

    @property
    def nnz(self):
        raise NotImplementedError


class Elimination(BlockOperator):
    """Block-Cholesky elimination of an interior (reference `:78-117`).

    ``panel_views`` is a list of (MatView, row0): consecutive row slices of
    the (|w_dofs| x |dofs|) panel; ``linv`` the explicit inverse of
    ``lower`` used by the apply (reference `tri_inverse`, dense.py:85-93).
    """

    kind = OpKind.ELIMINATION

    def __init__(self, dofs, w_dofs, lower, panel, linv=None):
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self._w_dofs = w_dofs if callable(w_dofs) else np.asarray(w_dofs, dtype=np.int64)
        self._lower = lower
        self._panel = panel if (isinstance(panel, list) or callable(panel)) else None
        self._panel_host = None if self._panel is not None else panel
        self.linv_view = linv

    @property
    def w_dofs(self):
        if callable(self._w_dofs):
            self._w_dofs = np.asarray(self._w_dofs(), dtype=np.int64)
        return self._w_dofs

    @property
    def lower(self):
        return _as_host(self._lower)

    @property
    def panel(self):
        if self._panel_host is None:
            ns = self.dofs.size
            views = self.panel_views
            if not views:
                self._panel_host = np.zeros((self.w_dofs.size, ns))
            else:
                self._panel_host = np.vstack([v.host() for v, _ in views])
        return self._panel_host

    @property
    def panel_views(self):
        if callable(self._panel):
            self._panel = self._panel()
        return self._panel

    @property
    def nnz(self):
        low = (self._lower.count_nonzero() if isinstance(self._lower, MatView)
               else int(np.count_nonzero(self._lower)))
        if self._panel is not None:
            pan = sum(v.count_nonzero() for v, _ in self.panel_views)
        else:
            pan = int(np.count_nonzero(self._panel_host))
        return int(low + pan)


class Scaling(BlockOperator):
    """Rescaling of an interface block to the identity (reference `:120-144`)."""

    kind = OpKind.SCALING

    def __init__(self, dofs, lower, linv=None):
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self._lower = lower
        self.linv_view = linv

    @property
    def lower(self):
        return _as_host(self._lower)

    @property
    def nnz(self):
        if isinstance(self._lower, MatView):
            return self._lower.count_nonzero()
        return int(np.count_nonzero(self._lower))


class Orthogonal(BlockOperator):
    """Orthogonal change of basis, columns fine-first (reference `:147-170`)."""

    kind = OpKind.ORTHOGONAL

    def __init__(self, dofs, q):
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self._q = q

    @property
    def q(self):
        return _as_host(self._q)

    @property
    def q_view(self):
        return self._q

    @property
    def nnz(self):
        if isinstance(self._q, MatView):
            return self._q.count_nonzero()
        return int(np.count_nonzero(self._q))


class ErrorCorrection(BlockOperator):
    """Second-order correction (reference `:173-196`).

    ``e_views`` is a list of (MatView, col0): consecutive column slices of
    the (|dofs| x |w_dofs|) correction block.
    """

    kind = OpKind.ERROR_CORRECTION

    def __init__(self, dofs, w_dofs, e_tilde):
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self._w_dofs = w_dofs if callable(w_dofs) else np.asarray(w_dofs, dtype=np.int64)
        self._e = e_tilde if (isinstance(e_tilde, list) or callable(e_tilde)) else None
        self._e_host = None if self._e is not None else e_tilde

    @property
    def w_dofs(self):
        if callable(self._w_dofs):
            self._w_dofs = np.asarray(self._w_dofs(), dtype=np.int64)
        return self._w_dofs

    @property
    def e_tilde(self):
        if self._e_host is None:
            self._e_host = np.hstack([v.host() for v, _ in self.e_views])
        return self._e_host

    @property
    def e_views(self):
        if callable(self._e):
            self._e = self._e()
        return self._e

    @property
    def nnz(self):
        if self._e is not None:
            return int(sum(v.count_nonzero() for v, _ in self.e_views))
        return int(np.count_nonzero(self._e_host))


# ---------------------------------------------------------------------------
# single-block constructors (reference schemes.py:199-340), on the device
# kernels through dense.py; the factorization itself batches these steps
# (engine.py), these are the per-block API of the reference.


def make_elimination(a_ss, a_ws, s_dofs=None, w_dofs=None):
    """Eliminate an interior block by one step of block Cholesky (reference
    `schemes.py:199-221`): returns (Elimination, Schur update panel panel^T)."""
    from . import kernels
    from .dense import cholesky, tri_solve
    a_ss = np.asarray(a_ss, dtype=np.float64)
    a_ws = np.asarray(a_ws, dtype=np.float64)
    ns, nw = a_ss.shape[0], a_ws.shape[0]
    s_dofs = np.arange(ns) if s_dofs is None else s_dofs
    w_dofs = ns + np.arange(nw) if w_dofs is None else w_dofs
    lower = cholesky(a_ss)
    if nw:
        panel = tri_solve(lower, a_ws, trans=True, side="right")
        update = kernels.gemm_one(panel, panel, trans_b=True)
    else:
        panel = np.zeros((0, ns))
        update = np.zeros((0, 0))
    return Elimination(s_dofs, w_dofs, lower, panel), update


def make_scaling(a_pp, a_pw, p_dofs=None):
    """Rescale an interface block to the identity (reference
    `schemes.py:224-236`): returns (Scaling, Z^-1 A_pw)."""
    from .dense import cholesky, tri_solve
    a_pp = np.asarray(a_pp, dtype=np.float64)
    a_pw = np.asarray(a_pw, dtype=np.float64)
    p_dofs = np.arange(a_pp.shape[0]) if p_dofs is None else p_dofs
    lower = cholesky(a_pp)
    panel = tri_solve(lower, a_pw) if a_pw.size else np.zeros(a_pw.shape)
    return Scaling(p_dofs, lower), panel


def _spectral(a):
    """Largest singular value on the device (sqrt of the top eigenvalue of
    the smaller Gram matrix)."""
    from .device import require_cuda, dev
    if min(a.shape) == 0:
        return 0.0
    t = require_cuda()
    m = t.as_tensor(np.ascontiguousarray(a), dtype=t.float64, device=dev())
    g = m @ m.t() if m.shape[0] <= m.shape[1] else m.t() @ m
    return float(t.linalg.eigvalsh(g)[-1].clamp_min(0).sqrt().item())


@dataclass(frozen=True)
class SparsificationResult:
    """Operators and bookkeeping of one sparsification (reference
    `schemes.py:245-269`)."""

    orthogonal: "Orthogonal"
    correction: "ErrorCorrection | None"
    coarse_rows: np.ndarray
    n_fine: int
    rank_c: int
    rank_f2: int
    scheme: object
    e_norm: float | None = field(default=None)
    e1_norm: float | None = field(default=None)
    e2_norm: float | None = field(default=None)


def make_sparsification(panel, eps, scheme, p_dofs=None, w_dofs=None,
                        keep_error_info=True):
    """Compress one rescaled interface panel (reference `schemes.py:272-318`)
    with the device RRQR; dropped-term norms on request."""
    from .dense import SchemeKind, rrqr_sparsify
    if isinstance(scheme, str):
        scheme = SchemeKind.from_string(scheme)
    panel = np.asarray(panel, dtype=np.float64)
    m, nw = panel.shape
    p_dofs = np.arange(m) if p_dofs is None else np.asarray(p_dofs)
    w_dofs = m + np.arange(nw) if w_dofs is None else w_dofs
    res = rrqr_sparsify(panel, eps, scheme)
    n_fine = m - res.rank_c
    orthogonal = Orthogonal(p_dofs, np.hstack([res.q_f, res.q_c]))
    n_corr = res.e_tilde.shape[0]
    correction = None
    if n_corr and res.e_tilde.size:
        correction = ErrorCorrection(p_dofs[:n_corr], w_dofs, res.e_tilde)
    e_norm = e1_norm = e2_norm = None
    if keep_error_info:
        from . import kernels
        if scheme is SchemeKind.SECOND_ORDER_SUPERFINE:
            e2_norm = _spectral(res.e_tilde)
            q_f1 = res.q_f[:, res.rank_f2:]
            e1_norm = (_spectral(kernels.gemm_one(q_f1, panel, trans_a=True))
                       if q_f1.size else 0.0)
        elif scheme is SchemeKind.SECOND_ORDER_FULL:
            e_norm = _spectral(res.e_tilde)
        else:
            e_norm = (_spectral(kernels.gemm_one(res.q_f, panel, trans_a=True))
                      if res.q_f.size else 0.0)
    return SparsificationResult(orthogonal, correction, res.r_coarse, n_fine, res.rank_c,
                                res.rank_f2, scheme, e_norm, e1_norm, e2_norm)


def local_error(scheme, result):
    """Spectral norm of the exactly dropped term (reference
    `schemes.py:321-340`)."""
    from .dense import SchemeKind
    if isinstance(scheme, str):
        scheme = SchemeKind.from_string(scheme)
    if scheme is SchemeKind.FIRST_ORDER:
        if result.e_norm is None:
            raise ValueError("sparsification ran without error info")
        return result.e_norm
    if scheme is SchemeKind.SECOND_ORDER_FULL:
        if result.e_norm is None:
            raise ValueError("sparsification ran without error info")
        return result.e_norm ** 2
    if scheme is SchemeKind.SECOND_ORDER_SUPERFINE:
        if result.e1_norm is None or result.e2_norm is None:
            raise ValueError("sparsification ran without error info")
        return max(result.e2_norm ** 2, result.e1_norm)
    raise ValueError(f"unknown scheme {scheme!r}")
