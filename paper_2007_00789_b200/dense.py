"""Dense kernel API of the reference (`dense.py:21-222`) on the B200.

``SchemeKind`` is unchanged.  ``cholesky``, ``tri_solve``, ``tri_inverse``
and ``rrqr_sparsify`` keep the reference signatures and error behaviour but
run the batched sm_100a kernels on a batch of one (the factorization itself
calls the batched entry points directly, a whole level per launch).
"""

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import DimensionMismatch, NonFinite, NotSPD, SingularTriangular


class SchemeKind(Enum):
    """Off-diagonal sparsification schemes (reference `dense.py:21-42`)."""

    FIRST_ORDER = "first"
    SECOND_ORDER_FULL = "second-full"
    SECOND_ORDER_SUPERFINE = "second-superfine"

    @classmethod
    def from_string(cls, s):
        for kind in cls:
            if kind.value == s:
                return kind
        names = ", ".join(k.value for k in cls)
        raise ValueError(f"unknown scheme {s!r} (expected one of: {names})")


SCHEME_CODE = {SchemeKind.FIRST_ORDER: 0, SchemeKind.SECOND_ORDER_FULL: 1,
               SchemeKind.SECOND_ORDER_SUPERFINE: 2}


@dataclass(frozen=True)
class RRQRResult:
    """Outcome of the early-stopping pivoted QR (reference `dense.py:96-114`)."""

    perm: np.ndarray
    q_c: np.ndarray
    q_f: np.ndarray
    r_coarse: np.ndarray
    e_tilde: np.ndarray
    rank_c: int
    rank_f2: int


def _square(m, what):
    a = np.asarray(m, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionMismatch(f"{what} needs a square matrix")
    return a


def cholesky(m):
    """Lower Cholesky factor on the GPU; NotSPD(pivot) on failure."""
    from . import kernels
    a = _square(m, "cholesky")
    if a.shape[0] == 0:
        return np.zeros((0, 0))
    l, info = kernels.potrf_one(a)
    if info > 0:
        raise NotSPD(info - 1)
    return l


def tri_inverse(l):
    """Explicit inverse of a lower-triangular factor on the GPU."""
    from . import kernels
    l = _square(l, "tri_inverse")
    if l.shape[0] == 0:
        return np.zeros((0, 0))
    d = np.diag(l)
    zero = np.flatnonzero(d == 0.0)
    if zero.size:
        raise SingularTriangular(zero[0])
    return kernels.trtri_one(l)


def tri_solve(l, b, trans=False, side="left"):
    """L X = B / L^T X = B (left) or X L = B / X L^T = B (right), on the GPU
    as a product with the explicit inverse (the factorization's TRSM)."""
    from . import kernels
    l = np.asarray(l, dtype=np.float64)
    zero = np.flatnonzero(np.abs(np.diag(l)) == 0.0)
    if zero.size:
        raise SingularTriangular(zero[0])
    if side not in ("left", "right"):
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    b = np.asarray(b, dtype=np.float64)
    vec = b.ndim == 1
    b2 = b.reshape(-1, 1) if vec else b
    if side == "right" and vec:
        b2 = b.reshape(1, -1)
    linv = kernels.trtri_one(l) if l.shape[0] else np.zeros((0, 0))
    # left:  X = L^-1 B  or  L^-T B ; right: X = B L^-1 or B L^-T
    if side == "left":
        x = kernels.gemm_one(linv, b2, trans_a=trans, trans_b=False)
    else:
        x = kernels.gemm_one(b2, linv, trans_a=False, trans_b=trans)
    return x.reshape(b.shape)


def rrqr_sparsify(a_pw, eps, scheme):
    """Rank-revealing QR of one panel with the scheme's stopping rules
    (reference `dense.py:186-222`), on the GPU RRQR kernel."""
    from . import kernels
    a = np.array(a_pw, dtype=np.float64, copy=True)
    if a.ndim != 2:
        raise DimensionMismatch("panel must be 2-D")
    if not np.all(np.isfinite(a)):
        raise NonFinite("panel contains NaN or Inf")
    if not 0.0 <= eps <= 1.0:
        raise ValueError(f"eps must lie in [0, 1], got {eps}")
    if isinstance(scheme, str):
        scheme = SchemeKind.from_string(scheme)
    return kernels.rrqr_one(a, eps, scheme)
