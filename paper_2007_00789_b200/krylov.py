"""Preconditioned conjugate gradients on the B200 (reference `krylov.py`).

Same contract as the reference `pcg` (`krylov.py:73-137`): zero initial
guess, recursively updated residual, strict ``rel < tol`` stop, history
entry 0 equal to 1.0, ``Breakdown`` when r.z <= 0 or p.Ap <= 0,
``converged=False`` at ``maxit``, and a final true residual.

The vectors live on the device.  When ``a`` is a ``SparseSymMatrix`` and
``m`` a factor (or its ``apply_m``), every step runs on the GPU: CSR SpMV
with a fused p.Ap partial, fused x/r update with an r.r partial, the batched
factor apply, deterministic two-stage dots.  One small device->host read
per iteration carries (p.Ap, r.r, r.z) for the stopping and breakdown tests;
the preconditioner step of the next iteration is issued before that read so
the host round trip overlaps device work.  Other operator kinds (callables,
objects with ``matvec``, dense arrays) are honoured as in the reference;
host callables get host vectors.
"""

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import dev, ptr, require_cuda, stream
from .errors import Breakdown

__all__ = ["SolveReport", "pcg", "cg_bound_rate", "default_maxit"]


@dataclass
class SolveReport:
    n_cg: int
    residual_history: list
    converged: bool
    true_residual: float
    solve_seconds: float
    eps: float | None = None
    scheme: str | None = None
    mu: float | None = None
    factor_seconds: float | None = None

    def as_dict(self):
        return {
            "n_cg": self.n_cg,
            "residual_history": list(self.residual_history),
            "converged": self.converged,
            "true_residual": self.true_residual,
            "solve_seconds": self.solve_seconds,
            "eps": self.eps,
            "scheme": self.scheme,
            "mu": self.mu,
            "factor_seconds": self.factor_seconds,
        }


def default_maxit(n):
    """int(10 sqrt(n) + 100) (reference `krylov.py:68-70`)."""
    return int(10.0 * math.sqrt(n) + 100.0)


def cg_bound_rate(kappa):
    """Asymptotic CG contraction factor for condition number kappa."""
    if kappa < 1.0:
        raise ValueError(f"condition number must be at least 1, got {kappa}")
    root = math.sqrt(kappa)
    return (root - 1.0) / (root + 1.0)


def _device_operator(op, n, what):
    """Return f(xd, out) writing op(x) into the device tensor ``out``."""
    t = require_cuda()
    from .factorize import Factorization
    from .sparse import SparseSymMatrix
    if op is None:
        return lambda xd, out: out.copy_(xd)
    target = getattr(op, "__self__", None)
    if isinstance(op, Factorization) or (
            isinstance(target, Factorization)
            and getattr(op, "__name__", "") == "apply_m"):
        fac = op if isinstance(op, Factorization) else target

        def run_m(xd, out):
            out.copy_(xd)
            fac.apply_m_device(out)
            return out
        return run_m
    if isinstance(op, SparseSymMatrix) or (
            isinstance(target, SparseSymMatrix)
            and getattr(op, "__name__", "") in ("matvec", "__matmul__")):
        mat = (op if isinstance(op, SparseSymMatrix) else target).device()
        return lambda xd, out: mat.spmv(xd, out)
    if callable(op) and not isinstance(op, np.ndarray):
        fn = op
    elif hasattr(op, "matvec"):
        fn = op.matvec
    else:
        arr = np.asarray(op, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise ValueError(f"{what} must be square, got shape {arr.shape}")
        dense = t.from_numpy(np.ascontiguousarray(arr)).to(dev())
        return lambda xd, out: out.copy_(dense @ xd)

    def host_call(xd, out):
        y = fn(xd.cpu().numpy())
        out.copy_(t.as_tensor(np.asarray(y, dtype=np.float64)).to(dev()))
        return out
    return host_call


class _Dots:
    """Deterministic device dot products into a small scalar array."""

    def __init__(self, n):
        t = require_cuda()
        lib = _lib.load()
        self.n = n
        self.nb = max(1, lib.spand_dot_blocks(n))
        self.part = t.empty(max(self.nb, lib.spand_spmv_blocks(n), 1),
                            dtype=t.float64, device=dev())

    def dot(self, x, y, out_slot):
        _lib.call("spand_dot", self.n, ptr(x), ptr(y), ptr(self.part),
                  ptr(out_slot), stream())


def pcg(a, b, m=None, tol=1e-10, maxit=None):
    """Solve A x = b by PCG on the device; returns (x, SolveReport)."""
    if tol <= 0.0:
        raise ValueError(f"tol must be positive, got {tol}")
    t = require_cuda()
    from .sparse import SparseSymMatrix
    is_torch = isinstance(b, t.Tensor)
    bd = (b.to(device=dev(), dtype=t.float64).contiguous() if is_torch
          else t.from_numpy(np.array(b, dtype=np.float64)).to(dev()))
    n = int(bd.shape[0])
    if maxit is None:
        maxit = default_maxit(n)
    lib = _lib.load()
    st = stream()
    spmv_mat = None
    if isinstance(a, SparseSymMatrix):
        spmv_mat = a.device()
    elif isinstance(getattr(a, "__self__", None), SparseSymMatrix):
        spmv_mat = a.__self__.device()
    apply_a = _device_operator(a, n, "system operator")
    apply_m = _device_operator(m, n, "preconditioner")
    dots = _Dots(n)
    scal = t.zeros(8, dtype=t.float64, device=dev())   # rz pap rz' rr bb
    start = time.perf_counter()
    x = t.zeros(n, dtype=t.float64, device=dev())

    def back(xo):
        return xo.to(b.device) if is_torch else xo.cpu().numpy()

    dots.dot(bd, bd, scal[4:5])
    b_norm = math.sqrt(float(scal[4].item()))
    if b_norm == 0.0:
        from .krylov import SolveReport as _SR  # noqa: F401
        return back(x), SolveReport(n_cg=0, residual_history=[0.0],
                                    converged=True, true_residual=0.0,
                                    solve_seconds=time.perf_counter() - start)
    r = bd.clone()
    z = t.empty_like(r)
    ap = t.empty_like(r)
    history = [1.0]
    apply_m(r, z)
    dots.dot(r, z, scal[0:1])
    rz = float(scal[0].item())
    if rz <= 0.0:
        raise Breakdown(f"preconditioner is not positive definite (r'z = {rz})")
    p = z.clone()
    converged = False
    iterations = 0
    nsp = max(1, lib.spand_spmv_blocks(n))
    for k in range(1, maxit + 1):
        if spmv_mat is not None:
            spmv_mat.spmv(p, ap, pdot=dots.part)
            _lib.call("spand_reduce_sum", nsp, ptr(dots.part), ptr(scal[1:2]), st)
        else:
            apply_a(p, ap)
            dots.dot(p, ap, scal[1:2])
        _lib.call("spand_pcg_xr", n, ptr(scal), ptr(x), ptr(r), ptr(p), ptr(ap),
                  ptr(dots.part), st)
        _lib.call("spand_reduce_sum", dots.nb, ptr(dots.part), ptr(scal[3:4]), st)
        # speculative preconditioner step for iteration k+1 (x, r untouched)
        apply_m(r, z)
        dots.dot(r, z, scal[2:3])
        vals = scal[:4].cpu().numpy()
        pap, rr, rz_next = float(vals[1]), float(vals[3]), float(vals[2])
        if pap <= 0.0:
            raise Breakdown(f"system operator is not positive definite "
                            f"(p'Ap = {pap})")
        rel = math.sqrt(max(rr, 0.0)) / b_norm
        history.append(rel)
        iterations = k
        if rel < tol:
            converged = True
            break
        if rz_next <= 0.0:
            raise Breakdown(f"preconditioner is not positive definite "
                            f"(r'z = {rz_next})")
        _lib.call("spand_pcg_p", n, ptr(scal), ptr(z), ptr(p), st)
        scal[0:1].copy_(scal[2:3])
    apply_a(x, ap)
    ap.sub_(bd).neg_()
    dots.dot(ap, ap, scal[5:6])
    true_residual = math.sqrt(float(scal[5].item())) / b_norm
    report = SolveReport(n_cg=iterations, residual_history=history,
                         converged=converged, true_residual=true_residual,
                         solve_seconds=time.perf_counter() - start)
    return back(x), report
