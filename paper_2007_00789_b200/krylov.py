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

__all__ = ["SolveReport", "pcg", "pcg_multi", "cg_bound_rate", "default_maxit"]


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
    """Solve A x = b by PCG on the device; returns (x, SolveReport).

    ``b`` of shape (n, k) (EXTENSION): k right-hand sides
    solved together (``pcg_multi``); returns (X, [SolveReport] * k)."""
    from .device import nvtx
    with nvtx("spand.pcg"):
        return _pcg_impl(a, b, m, tol, maxit)


def _pcg_impl(a, b, m=None, tol=1e-10, maxit=None):
    """Solve A x = b by PCG on the device; returns (x, SolveReport).

    ``b`` of shape (n, k) (EXTENSION): k right-hand sides
    solved together (``pcg_multi``); returns (X, [SolveReport] * k)."""
    if tol <= 0.0:
        raise ValueError(f"tol must be positive, got {tol}")
    t = require_cuda()
    if getattr(b, "ndim", 1) == 2:
        return pcg_multi(a, b, m=m, tol=tol, maxit=maxit)
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


def _rows_apply(m, n):
    """Preconditioner on a contiguous (k, n) stack of row vectors, in place:
    a device factor runs its multi-RHS apply (each payload element read once
    per group of up to four vectors, every row bitwise equal to the
    single-vector apply); other operators run row by row."""
    from .factorize import Factorization
    target = getattr(m, "__self__", None)
    fac = m if isinstance(m, Factorization) else (
        target if isinstance(target, Factorization)
        and getattr(m, "__name__", "") == "apply_m" else None)
    if fac is not None:
        plan = fac.plan
        if hasattr(plan, "run_rows"):
            return lambda rows: plan.run_rows(rows)

        def cols_run(rows):
            cols = rows.t().contiguous()
            plan.run(cols)
            rows.copy_(cols.t())
            return rows
        return cols_run
    single = _device_operator(m, n, "preconditioner")

    def each(rows):
        t = require_cuda()
        tmp = t.empty(n, dtype=t.float64, device=dev())
        for j in range(rows.shape[0]):
            single(rows[j], tmp)
            rows[j].copy_(tmp)
        return rows
    return each


def pcg_multi(a, b, m=None, tol=1e-10, maxit=None):
    """k right-hand sides by PCG in lockstep (multi-RHS solve, SURVEY 8f-3,
    the column stacks of factorize.py:262-267): every column runs exactly
    the recurrence of ``pcg`` -- same kernels, same order, so each column's
    iterates, history and stopping decision are bit for bit those of a
    single-vector solve -- while the preconditioner applies to the stack of
    still-running columns at once.  Returns (X (n, k), [SolveReport] * k)."""
    if tol <= 0.0:
        raise ValueError(f"tol must be positive, got {tol}")
    t = require_cuda()
    from .sparse import SparseSymMatrix
    is_torch = isinstance(b, t.Tensor)
    bd = (b.to(device=dev(), dtype=t.float64) if is_torch
          else t.from_numpy(np.array(b, dtype=np.float64)).to(dev()))
    if bd.dim() != 2:
        raise ValueError("pcg_multi needs an (n, k) right-hand side")
    n, k = int(bd.shape[0]), int(bd.shape[1])
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
    apply_rows = _rows_apply(m, n)
    dots = [_Dots(n) for _ in range(k)]
    nsp = max(1, lib.spand_spmv_blocks(n))
    scal = t.zeros((k, 8), dtype=t.float64, device=dev())
    start = time.perf_counter()
    B = bd.t().contiguous()                       # (k, n): rows are the systems
    X = t.zeros_like(B)
    R = B.clone()
    Z = t.empty_like(B)
    P = t.empty_like(B)
    AP = t.empty_like(B)
    for j in range(k):
        dots[j].dot(B[j], B[j], scal[j, 4:5])
    bnorm = np.sqrt(scal[:, 4].cpu().numpy())
    hist = [[1.0] if bnorm[j] > 0 else [0.0] for j in range(k)]
    live = [j for j in range(k) if bnorm[j] > 0]
    iters = [0] * k
    conv = [bnorm[j] == 0 for j in range(k)]

    def precond(rows_idx):
        # Z[j] = M R[j] for the given rows, as one stack
        if not rows_idx:
            return
        if len(rows_idx) == k:
            Z.copy_(R)
            apply_rows(Z)
            return
        idx = t.as_tensor(rows_idx, device=dev())
        stack = R.index_select(0, idx).contiguous()
        apply_rows(stack)
        Z.index_copy_(0, idx, stack)

    precond(live)
    for j in live:
        dots[j].dot(R[j], Z[j], scal[j, 0:1])
    rz = scal[:, 0].cpu().numpy()
    for j in live:
        if rz[j] <= 0.0:
            raise Breakdown(f"preconditioner is not positive definite "
                            f"(column {j}: r'z = {rz[j]})")
    P.copy_(Z)
    for it in range(1, maxit + 1):
        if not live:
            break
        for j in live:
            if spmv_mat is not None:
                spmv_mat.spmv(P[j], AP[j], pdot=dots[j].part)
                _lib.call("spand_reduce_sum", nsp, ptr(dots[j].part), ptr(scal[j, 1:2]), st)
            else:
                apply_a(P[j], AP[j])
                dots[j].dot(P[j], AP[j], scal[j, 1:2])
            _lib.call("spand_pcg_xr", n, ptr(scal[j]), ptr(X[j]), ptr(R[j]), ptr(P[j]),
                      ptr(AP[j]), ptr(dots[j].part), st)
            _lib.call("spand_reduce_sum", dots[j].nb, ptr(dots[j].part), ptr(scal[j, 3:4]), st)
        precond(live)
        for j in live:
            dots[j].dot(R[j], Z[j], scal[j, 2:3])
        vals = scal[:, :4].cpu().numpy()
        still = []
        for j in live:
            pap, rr, rz_next = float(vals[j, 1]), float(vals[j, 3]), float(vals[j, 2])
            if pap <= 0.0:
                raise Breakdown(f"system operator is not positive definite "
                                f"(column {j}: p'Ap = {pap})")
            rel = math.sqrt(max(rr, 0.0)) / bnorm[j]
            hist[j].append(rel)
            iters[j] = it
            if rel < tol:
                conv[j] = True
                continue
            if rz_next <= 0.0:
                raise Breakdown(f"preconditioner is not positive definite "
                                f"(column {j}: r'z = {rz_next})")
            _lib.call("spand_pcg_p", n, ptr(scal[j]), ptr(Z[j]), ptr(P[j]), st)
            scal[j, 0:1].copy_(scal[j, 2:3])
            still.append(j)
        live = still
    reports = []
    for j in range(k):
        if bnorm[j] == 0:
            tres = 0.0
        else:
            apply_a(X[j], AP[j])
            AP[j].sub_(B[j]).neg_()
            dots[j].dot(AP[j], AP[j], scal[j, 5:6])
            tres = math.sqrt(float(scal[j, 5].item())) / bnorm[j]
        reports.append(SolveReport(n_cg=iters[j], residual_history=hist[j],
                                   converged=bool(conv[j]), true_residual=tres,
                                   solve_seconds=time.perf_counter() - start))
    Xo = X.t().contiguous()
    return (Xo.to(b.device) if is_torch else Xo.cpu().numpy()), reports
