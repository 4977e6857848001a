"""Factorization object, factor I/O and the public ``factorize`` entry point.

API of the reference `factorize.py:242-502`: ``Factorization`` (ops, perm,
n, eps, scheme, skip_levels, nnz_factor, diagnostics, apply_inv /
apply_inv_t / apply_m), ``factorize``, ``apply_inv``, ``apply_inv_t``,
``memory_ratio``, ``save_factor`` / ``load_factor`` (the "SPDF" v1 container,
byte-compatible with the reference's files).

The numerical work of ``factorize`` is the device engine in ``engine.py``;
the apply is the batched device plan of ``apply.py``.  Inputs and outputs
of ``apply_*`` may be NumPy arrays (copied to and from the device) or CUDA
tensors (kept on the device).
"""

import struct
from dataclasses import dataclass, field

import numpy as np

from .dense import SchemeKind
from .device import as_device_vector, like_input, require_cuda, to_dev
from .errors import DimensionMismatch, ParseError
from .schemes import (Elimination, ErrorCorrection, MatView, OpKind, Orthogonal,
                      Scaling)

__all__ = ["Factorization", "factorize", "apply_inv", "apply_inv_t",
           "memory_ratio", "save_factor", "load_factor"]


@dataclass
class Factorization:
    """Completed factor: an ordered list of block operators (device payloads)."""

    ops: list
    perm: np.ndarray
    n: int
    eps: float
    scheme: SchemeKind
    skip_levels: int
    nnz_factor: int
    diagnostics: dict | None = field(default=None, repr=False)
    _plan: object = field(default=None, repr=False, compare=False)
    _keep: object = field(default=None, repr=False, compare=False)
    timings: dict | None = field(default=None, repr=False, compare=False)
    _plan_factory: object = field(default=None, repr=False, compare=False)

    @property
    def plan(self):
        """Device apply plan: the structured fast plan for factors built by
        the engine, the generic scheduled plan for loaded factors."""
        if self._plan is None:
            if self._plan_factory is not None:
                self._plan = self._plan_factory()
            else:
                from .apply import ApplyPlan
                self._plan = ApplyPlan(self.n, self.ops)
        return self._plan

    def _run(self, x, fwd, bwd):
        xd, kind = as_device_vector(x, self.n)
        self.plan.run(xd, forward=fwd, backward=bwd)
        return like_input(xd, kind)

    def apply_inv(self, x):
        return self._run(x, True, False)

    def apply_inv_t(self, x):
        return self._run(x, False, True)

    def apply_m(self, x):
        return self._run(x, True, True)

    def apply_m_device(self, xd):
        """In-place M x on a contiguous fp64 CUDA vector (graph replay)."""
        if xd.dim() == 1:
            return self.plan.run_graph(xd)
        return self.plan.run(xd)


def apply_inv(factor, x):
    return factor.apply_inv(x)


def apply_inv_t(factor, x):
    return factor.apply_inv_t(x)


def memory_ratio(factor, a):
    """Stored factor nonzeros relative to nnz(A) (reference `:379-381`)."""
    return factor.nnz_factor / a.nnz


def factorize(a, hierarchy, eps, scheme, skip_levels=4,
              collect_local_errors=False, near_kernel=None, digest=True):
    """Factor a sparse SPD matrix over a partition hierarchy on the B200.

    Same contract as the reference (`factorize.py:285-366`): levels from the
    finest to the coarsest, interiors eliminated, then (outside the first
    ``skip_levels`` levels) every active interface rescaled and sparsified
    in ascending id order; the leftover clusters form one dense block.
    ``near_kernel`` (EXTENSION, off by default; not in the reference): an
    n-vector or n x k array (k <= 16) of near-kernel vectors, e.g. the
    constant vector or rigid-body modes.  Each sparsification then keeps the
    vectors' restriction to the interface (carried through the factor's
    congruences) inside the coarse basis, so the preconditioner stays
    accurate on them.  None or k = 0 is the reference path exactly.
    """
    if isinstance(scheme, str):
        scheme = SchemeKind.from_string(scheme)
    if not 0.0 <= eps <= 1.0:
        raise ValueError(f"eps must lie in [0, 1], got {eps}")
    if skip_levels < 0:
        raise ValueError(f"skip_levels must be nonnegative, got {skip_levels}")
    if a.n != hierarchy.n:
        raise DimensionMismatch(
            f"matrix has {a.n} dofs but hierarchy covers {hierarchy.n}")
    nk = None
    if near_kernel is not None:
        nk = np.asarray(near_kernel, dtype=np.float64)
        if nk.ndim not in (1, 2) or nk.shape[0] != a.n:
            raise DimensionMismatch(
                f"near_kernel must have {a.n} rows, got shape {nk.shape}")
        nk = nk.reshape(a.n, -1)
        if nk.shape[1] > 16:
            raise ValueError(f"at most 16 near-kernel vectors, got {nk.shape[1]}")
        if nk.shape[1] == 0:
            nk = None
    from .engine import check_panel_rows, run_factorization
    check_panel_rows(hierarchy, int(skip_levels))
    return run_factorization(a, hierarchy, float(eps), scheme, int(skip_levels),
                             collect_local_errors, near_kernel=nk, digest=bool(digest))


# ---------------------------------------------------------------------------
# SPDF v1 container (reference `factorize.py:384-502`)

_MAGIC = b"SPDF"
_VERSION = 1
_HDR = "<HqdBHIq"
_KIND_TAG = {OpKind.ELIMINATION: 0, OpKind.SCALING: 1, OpKind.ORTHOGONAL: 2,
             OpKind.ERROR_CORRECTION: 3}
_SCHEME_TAG = {SchemeKind.FIRST_ORDER: 0, SchemeKind.SECOND_ORDER_FULL: 1,
               SchemeKind.SECOND_ORDER_SUPERFINE: 2}
_SCHEME_OF = {v: k for k, v in _SCHEME_TAG.items()}


def _put(fh, arr, dtype):
    arr = np.ascontiguousarray(arr, dtype=dtype)
    fh.write(struct.pack("<B", arr.ndim))
    fh.write(struct.pack(f"<{arr.ndim}q", *arr.shape))
    fh.write(arr.tobytes())


def _take(fh, count):
    data = fh.read(count)
    if len(data) != count:
        raise ParseError("truncated factor file")
    return data


def _get(fh, dtype):
    ndim = struct.unpack("<B", _take(fh, 1))[0]
    shape = struct.unpack(f"<{ndim}q", _take(fh, 8 * ndim))
    count = int(np.prod(shape)) if ndim else 1
    if count < 0:
        raise ParseError("negative array extent")
    data = _take(fh, count * np.dtype(dtype).itemsize)
    return np.frombuffer(data, dtype=dtype).reshape(shape).copy()


def save_factor(factor, path):
    """Write a factor (payloads streamed from the device) as SPDF v1."""
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack(_HDR, _VERSION, factor.n, factor.eps,
                             _SCHEME_TAG[factor.scheme], factor.skip_levels,
                             len(factor.ops), factor.nnz_factor))
        _put(fh, factor.perm, np.int64)
        for op in factor.ops:
            fh.write(struct.pack("<B", _KIND_TAG[op.kind]))
            _put(fh, op.dofs, np.int64)
            if op.kind is OpKind.ELIMINATION:
                _put(fh, op.w_dofs, np.int64)
                _put(fh, op.lower, np.float64)
                _put(fh, op.panel, np.float64)
            elif op.kind is OpKind.SCALING:
                _put(fh, op.lower, np.float64)
            elif op.kind is OpKind.ORTHOGONAL:
                _put(fh, op.q, np.float64)
            else:
                _put(fh, op.w_dofs, np.int64)
                _put(fh, op.e_tilde, np.float64)


class _Arena:
    """Packs host matrices column-major into one device buffer."""

    def __init__(self):
        self.parts, self.size = [], 0

    def add(self, arr):
        arr = np.asarray(arr, dtype=np.float64)
        at = self.size
        self.parts.append(np.ascontiguousarray(arr.T).ravel())
        self.size += arr.size
        return at

    def reserve(self, count):
        at = self.size
        self.parts.append(np.zeros(count))
        self.size += count
        return at

    def upload(self):
        return to_dev(np.concatenate(self.parts) if self.parts
                      else np.zeros(1))


def device_ops_from_host(raw_ops):
    """Upload host payloads and build device-backed operators.

    ``raw_ops`` are tuples (kind, dofs, w_dofs, payload dict).  Triangular
    inverses are computed on the device (batched trtri)."""
    from .kernels import Geometry, opnd, trtri_batched
    require_cuda()
    arena = _Arena()
    plan = []
    for kind, dofs, w_dofs, pay in raw_ops:
        ent = {"kind": kind, "dofs": dofs, "w_dofs": w_dofs}
        for name, arr in pay.items():
            ent[name] = (arena.add(arr), arr.shape)
        if kind in (OpKind.ELIMINATION, OpKind.SCALING):
            nsz = pay["lower"].shape[0]
            ent["linv"] = (arena.reserve(nsz * nsz), (nsz, nsz))
        plan.append(ent)
    buf = arena.upload()
    sizes, pairs = [], []
    ops = []
    for ent, (_, _, _, pay) in zip(plan, raw_ops):
        kind = ent["kind"]

        def view(name):
            at, shp = ent[name]
            v = MatView(buf, at, max(shp[0], 1), shp[0], shp[1])
            if name in pay:
                v._host = pay[name]
            return v

        if kind is OpKind.ELIMINATION:
            low, linv = view("lower"), view("linv")
            pv = view("panel")
            op = Elimination(ent["dofs"], ent["w_dofs"], low, [(pv, 0)],
                             linv=linv)
        elif kind is OpKind.SCALING:
            low, linv = view("lower"), view("linv")
            op = Scaling(ent["dofs"], low, linv=linv)
        elif kind is OpKind.ORTHOGONAL:
            op = Orthogonal(ent["dofs"], view("q"))
        else:
            op = ErrorCorrection(ent["dofs"], ent["w_dofs"], [(view("e_tilde"), 0)])
        if kind in (OpKind.ELIMINATION, OpKind.SCALING) and low.rows:
            cid = len(sizes)
            sizes.append(low.rows)
            pairs.append((opnd(low.addr, cid, cid), opnd(linv.addr, cid, cid)))
        ops.append(op)
    if pairs:
        geo = Geometry.virtual(sizes)
        trtri_batched(geo, pairs)
    return ops, buf


def load_factor(path):
    """Read an SPDF v1 factor (reference or ours) onto the device."""
    raw = []
    with open(path, "rb") as fh:
        if _take(fh, 4) != _MAGIC:
            raise ParseError("not a factor file (bad magic)")
        version, n, eps, stag, skip, nops, nnzf = struct.unpack(
            _HDR, _take(fh, struct.calcsize(_HDR)))
        if version != _VERSION:
            raise ParseError(f"unsupported factor file version {version}")
        if stag not in _SCHEME_OF:
            raise ParseError(f"unknown scheme tag {stag}")
        perm = _get(fh, np.int64)
        for _ in range(nops):
            tag = struct.unpack("<B", _take(fh, 1))[0]
            if tag == 0:
                dofs = _get(fh, np.int64)
                w = _get(fh, np.int64)
                raw.append((OpKind.ELIMINATION, dofs, w,
                            {"lower": _get(fh, np.float64),
                             "panel": _get(fh, np.float64)}))
            elif tag == 1:
                dofs = _get(fh, np.int64)
                raw.append((OpKind.SCALING, dofs, None,
                            {"lower": _get(fh, np.float64)}))
            elif tag == 2:
                dofs = _get(fh, np.int64)
                raw.append((OpKind.ORTHOGONAL, dofs, None,
                            {"q": _get(fh, np.float64)}))
            elif tag == 3:
                dofs = _get(fh, np.int64)
                w = _get(fh, np.int64)
                raw.append((OpKind.ERROR_CORRECTION, dofs, w,
                            {"e_tilde": _get(fh, np.float64)}))
            else:
                raise ParseError(f"unknown operator tag {tag}")
    ops, buf = device_ops_from_host(raw)
    return Factorization(ops=ops, perm=perm, n=int(n), eps=float(eps),
                         scheme=_SCHEME_OF[stag], skip_levels=int(skip),
                         nnz_factor=int(nnzf), diagnostics=None, _keep=buf)
