"""Block operators of the factor (reference `schemes.py:48-196`).

Same classes, kinds and attributes as the reference (``dofs``, ``w_dofs``,
``lower``, ``panel``, ``q``, ``e_tilde``, ``nnz``, ``apply_inv``,
``apply_inv_t``), but the payloads live on the B200: each attribute is a
``MatView`` (a window into a device buffer, column-major, possibly
transposed) materialised to NumPy only when a caller asks for it.  The
preconditioner never touches the host copies; it runs the batched apply
plan of ``apply.py`` on the device.
"""

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
