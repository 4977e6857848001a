"""Sparse symmetric matrices, BASELINE problem generators and Matrix Market I/O.

``SparseSymMatrix`` keeps the reference's constructor and invariants
(`/root/reference/pkg/src/spdkit/sparse.py:24-90`: CSR with both triangles,
strictly increasing columns, exact value symmetry, positive diagonal).  The
host arrays are the *input format*; every product of the matrix with a vector
(``matvec``/``@``) runs on the B200 through the C-ABI SpMV kernel
(``spand_csr_spmv``), with a device copy (int32 indices) uploaded lazily and
cached.  There is no host SpMV.

Generators:
- ``laplacian_2d`` reproduces the reference generator bit for bit
  (`sparse.py:181-196`; pinned by ``tests/golden``);
- ``laplacian_3d``, ``diffusion_fv`` and ``log_uniform_block_field`` build the
  BASELINE.json configs C2-C4 that the reference has no generator for
  (SURVEY.md §0, §8d): 7-point/5-point finite volumes, harmonic-mean face
  coefficients, Dirichlet boundary faces adding the cell's own coefficient
  (the reference's convention, `sparse.py:278-282`), so a constant field
  reduces exactly to the Laplacian.
- ``baseline_problem(name)`` returns (A, b, levels) for C1-C4 with the seeding
  convention "field first, then b = rng.standard_normal(n)".
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import (
    AsymmetricValues,
    DimensionMismatch,
    NonpositiveDiagonal,
    NotSymmetricReal,
    ParseError,
)


_CHECK_ERRORS = {1: (ParseError, "column index out of range"),
                 2: (ParseError, "column indices must be strictly increasing per row"),
                 3: (AsymmetricValues, "stored pattern or values are not symmetric"),
                 4: (NonpositiveDiagonal, "diagonal entries must be strictly positive")}


def _check_csr(n, rp, ci, va):
    """Range, order, exact symmetry and positive diagonal (reference
    `sparse.py:40-58`), first failing property raised: one native O(nnz log d)
    pass per property (csrc/validate.cpp)."""
    import ctypes
    from . import _lib
    lib = _lib.load()
    lib.spand_csr_check.restype = ctypes.c_int
    lib.spand_csr_check.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 3
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    va = np.ascontiguousarray(va, dtype=np.float64)
    code = lib.spand_csr_check(int(n), p(rp), p(ci), p(va))
    if code:
        err, msg = _CHECK_ERRORS[code]
        raise err(msg)


@dataclass(frozen=True)
class SparseSymMatrix:
    """Symmetric CSR matrix, both triangles stored (reference `sparse.py:24`)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    _dev: dict = field(repr=False, compare=False, default=None)

    def __post_init__(self):
        n = int(self.n)
        rp = np.asarray(self.row_ptr, dtype=np.int64)
        ci = np.asarray(self.col_idx, dtype=np.int64)
        va = np.asarray(self.values, dtype=np.float64)
        if rp.shape != (n + 1,):
            raise DimensionMismatch("row_ptr must have length n+1")
        counts = np.diff(rp)
        if np.any(counts < 1):
            raise NonpositiveDiagonal("every row needs its diagonal entry")
        if rp[0] != 0 or rp[-1] != ci.size or ci.size != va.size:
            raise DimensionMismatch("row_ptr, col_idx and values disagree")
        _check_csr(n, rp, ci, va)
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "row_ptr", rp)
        object.__setattr__(self, "col_idx", ci)
        object.__setattr__(self, "values", va)
        object.__setattr__(self, "_dev", {})

    @property
    def nnz(self):
        return int(self.values.size)

    def diagonal(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        d = np.zeros(self.n)
        m = rows == self.col_idx
        d[rows[m]] = self.values[m]
        return d

    def toarray(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        out = np.zeros((self.n, self.n))
        out[rows, self.col_idx] = self.values
        return out

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                             shape=(self.n, self.n))

    # -- device side -----------------------------------------------------
    def device(self, perm=None):
        """Device CSR (int32 indices, fp64 values), optionally symmetrically
        permuted so that new index ``i`` is old index ``perm[i]``."""
        from .device import DeviceCSR
        key = None if perm is None else id(perm)
        cached = self._dev.get(key)
        if cached is not None and (perm is None or cached[0] is perm):
            return cached[1]
        dev = DeviceCSR.from_host(self, perm)
        self._dev[key] = (perm, dev)
        return dev

    def matvec(self, x):
        """y = A x on the B200 (numpy in -> numpy out, torch in -> torch out)."""
        from .device import as_device_vector, like_input
        xd, kind = as_device_vector(x, self.n)
        y = self.device().spmv(xd)
        return like_input(y, kind)

    def __matmul__(self, x):
        return self.matvec(x)


def from_coo(n, rows, cols, vals):
    """SparseSymMatrix from COO triplets covering both triangles."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return SparseSymMatrix(n, row_ptr, cols, vals)


# ---------------------------------------------------------------------------
# Matrix Market (input side, reference `sparse.py:98-173`)


def read_matrix_market(path):
    """Read a `matrix coordinate real symmetric` file (one triangle stored),
    reference `sparse.py:98-160`: parsed by the native multi-threaded reader
    (csrc/mmio.cpp); the same errors, raised for the first offending line in
    file order, with the reference's messages."""
    import ctypes
    from . import _lib
    lib = _lib.load()
    lib.spand_mm_read.restype = ctypes.c_void_p
    lib.spand_mm_read.argtypes = [ctypes.c_char_p, ctypes.c_void_p]
    for nm, args in (("spand_mm_csr", 4), ("spand_mm_error_span", 2), ("spand_mm_text", 4)):
        getattr(lib, nm).argtypes = [ctypes.c_void_p] * args
        getattr(lib, nm).restype = ctypes.c_int
    lib.spand_mm_text.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_void_p]
    lib.spand_mm_free.argtypes = [ctypes.c_void_p]
    vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    info = np.zeros(8, dtype=np.int64)
    h = lib.spand_mm_read(str(path).encode(), vp(info))
    try:
        code = int(info[0])

        def text(b, e):
            buf = ctypes.create_string_buffer(max(int(e - b), 1))
            lib.spand_mm_text(h, int(b), int(e), buf)
            return buf.raw[:int(e - b)].decode(errors="replace")

        if code == 11:
            raise FileNotFoundError(path)
        if code in (1, 2, 3):
            header = text(0, info[5]).strip()
            tok = header.split()
            if code == 1:
                raise ParseError(f"bad Matrix Market header: {header!r}")
            if code == 2:
                raise ParseError(f"unsupported object/format: {header!r}")
            raise NotSymmetricReal(f"only real symmetric matrices are supported, got "
                                   f"{tok[3]} {tok[4]}")
        if code == 4:
            raise ParseError(f"bad size line: {text(info[6], info[7]).strip()!r}")
        if code == 5:
            raise NotSymmetricReal("matrix must be square")
        if code == 6:
            raise ParseError("file ends before declared entry count")
        if code:
            span = np.zeros(2, dtype=np.int64)
            lib.spand_mm_error_span(h, vp(span))
            line = text(span[0], span[1])
            if code == 7:
                raise ParseError(f"bad entry line: {line.strip()!r}")
            parts = line.split()
            i, j, v = int(parts[0]), int(parts[1]), float(parts[2])
            if code == 8:
                raise ParseError(f"index out of range: ({i}, {j})")
            if code == 9:
                raise ParseError(f"duplicate entry ({i}, {j})")
            mirror = float(np.int64(info[4]).view(np.float64))
            raise AsymmetricValues(f"entries ({j}, {i}) and ({i}, {j}) disagree: "
                                   f"{mirror} vs {v}")
        n, nnz = int(info[1]), int(info[2])
        rp = np.zeros(n + 1, dtype=np.int64)
        ci = np.zeros(max(nnz, 1), dtype=np.int64)
        va = np.zeros(max(nnz, 1), dtype=np.float64)
        lib.spand_mm_csr(h, vp(rp), vp(ci), vp(va))
    finally:
        lib.spand_mm_free(h)
    return SparseSymMatrix(n, rp, ci[:nnz], va[:nnz])


def write_matrix_market(path, a):
    """Write the lower triangle in coordinate format, column-major order."""
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    low = rows >= a.col_idx
    r, c, v = rows[low], a.col_idx[low], a.values[low]
    order = np.lexsort((r, c))
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n")
        fh.write(f"{a.n} {a.n} {r.size}\n")
        for k in order:
            fh.write(f"{r[k] + 1} {c[k] + 1} {v[k]:.17g}\n")


def jacobi_prescale(a, b, device=False):
    """A' = D^-1/2 A D^-1/2, b' = D^-1/2 b (reference `sparse.py:290-308`).

    ``device=True``: on the B200 (csrc/input.cu), bit for bit the same
    values; the scaled matrix keeps its device CSR cached.

    Input-side preprocessing (one pass over nnz(A)); the scale of entry
    (i, j) is the product s_i * s_j grouped the same way for (i, j) and
    (j, i) so the result stays exactly symmetric.
    """
    if device:
        return _jacobi_prescale_device(a, b)
    diag = a.diagonal()
    if np.any(diag <= 0.0):
        raise NonpositiveDiagonal("jacobi_prescale needs a positive diagonal")
    s = 1.0 / np.sqrt(diag)
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    vals = a.values * (s[rows] * s[a.col_idx])
    return (SparseSymMatrix(a.n, a.row_ptr, a.col_idx, vals),
            np.asarray(b, dtype=np.float64) * s, diag)


def _device_matrix(n, rp, ci, va):
    """SparseSymMatrix from device CSR arrays (int64 / fp64 tensors): host
    copies for the host-side structure (validation, partition), and the
    device CSR (int32 indices) cached so no host->device upload follows."""
    from .device import DeviceCSR, torch
    t = torch()
    a = SparseSymMatrix(int(n), rp.cpu().numpy(), ci.cpu().numpy(), va.cpu().numpy())
    a._dev[None] = (None, DeviceCSR(a.n, rp.to(t.int32), ci.to(t.int32), va))
    return a


def _jacobi_prescale_device(a, b):
    from . import _lib
    from .device import ptr, require_cuda, stream, to_dev
    t = require_cuda()
    n = a.n
    rp, ci = to_dev(a.row_ptr, np.int64), to_dev(a.col_idx, np.int64)
    va = to_dev(a.values, np.float64)
    diag = t.empty(n, dtype=t.float64, device=va.device)
    s = t.empty_like(diag)
    bd = to_dev(np.asarray(b, dtype=np.float64).copy(), np.float64)
    bad = t.zeros(1, dtype=t.int32, device=va.device)
    _lib.call("spand_jacobi_prescale", n, ptr(rp), ptr(ci), ptr(va), ptr(diag), ptr(s),
              ptr(bd), ptr(bad), stream())
    if int(bad.item()):
        raise NonpositiveDiagonal("jacobi_prescale needs a positive diagonal")
    return _device_matrix(n, rp, ci, va), bd.cpu().numpy(), diag.cpu().numpy()


def diffusion_fv_device(block_values, block, shape):
    """``diffusion_fv(field)`` for a piecewise-constant field (one value per
    block of ``block`` cells per axis, C order), generated on the B200
    (csrc/input.cu, bitwise equal to the host generator): the CSR is built in
    device memory and stays cached on the returned matrix."""
    from . import _lib
    from .device import ptr, require_cuda, stream, to_dev
    t = require_cuda()
    shape = tuple(int(x) for x in shape)
    bv = np.ascontiguousarray(block_values, dtype=np.float64)
    if len(shape) not in (2, 3) or min(shape) < 2:
        raise DimensionMismatch("need a 2D or 3D grid with sides >= 2")
    if bv.shape != tuple(x // block for x in shape) or any(
            (x // block) * block != x for x in shape):
        raise DimensionMismatch("grid must be a multiple of the block size")
    if np.any(bv <= 0.0):
        raise NonpositiveDiagonal("coefficients must be positive")
    n = int(np.prod(shape))
    dims = np.asarray(shape, dtype=np.int64)
    dptr = dims.ctypes.data
    import ctypes
    cnt = t.empty(n, dtype=t.int64, device="cuda")
    _lib.call("spand_fv_counts", len(shape), ctypes.c_void_p(dptr), ptr(cnt), stream())
    rp = t.zeros(n + 1, dtype=t.int64, device="cuda")
    t.cumsum(cnt, 0, out=rp[1:])
    nnz = int(rp[-1].item())
    ci = t.empty(nnz, dtype=t.int64, device="cuda")
    va = t.empty(nnz, dtype=t.float64, device="cuda")
    bvd = to_dev(bv.ravel(), np.float64)
    _lib.call("spand_fv_fill", len(shape), ctypes.c_void_p(dptr), int(block), ptr(bvd),
              ptr(rp), ptr(ci), ptr(va), stream())
    return _device_matrix(n, rp, ci, va)


# ---------------------------------------------------------------------------
# generators


def laplacian_2d(d):
    """5-point Laplacian on a d x d grid, Dirichlet, diagonal 4.

    Same matrix (index i*d+j, values 4/-1, sorted CSR) as the reference
    `sparse.py:181-196`.
    """
    if d < 2:
        raise DimensionMismatch("grid side must be at least 2")
    a = diffusion_fv(np.ones((d, d)))
    if d > 5:
        return a
    # For d <= 5 the reference's scipy kron takes its block-sparse path and
    # stores the d x d blocks of the block-tridiagonal pattern densely,
    # explicit zeros included; those zeros are graph edges for the
    # partitioner and count in nnz(A), so reproduce them.
    blk = np.arange(d * d) // d
    dense = a.toarray()
    rows, cols = np.nonzero(np.abs(blk[:, None] - blk[None, :]) <= 1)
    return from_coo(d * d, rows, cols, dense[rows, cols])


def laplacian_3d(d):
    """7-point Laplacian on a d^3 grid, Dirichlet, diagonal 6 (config C2)."""
    if d < 2:
        raise DimensionMismatch("grid side must be at least 2")
    return diffusion_fv(np.ones((d, d, d)))


def harmonic_face(a1, a2):
    """Harmonic mean 2 a1 a2 / (a1 + a2); exactly 1 for a1 = a2 = 1."""
    return 2.0 * a1 * a2 / (a1 + a2)


def diffusion_fv(coef):
    """Finite-volume -div(a grad u) on a 2D/3D cell grid, Dirichlet boundary.

    ``coef`` has one positive value per cell (shape (d0, d1) or (d0, d1, d2));
    cell index = C-order ravel.  Interior faces carry the harmonic mean of
    the two cells; a boundary face adds the cell's own coefficient to the
    diagonal.  Rows are emitted in CSR with sorted columns.
    """
    coef = np.asarray(coef, dtype=np.float64)
    if coef.ndim not in (2, 3) or min(coef.shape) < 2:
        raise DimensionMismatch("need a 2D or 3D grid with sides >= 2")
    if np.any(coef <= 0.0):
        raise NonpositiveDiagonal("coefficients must be positive")
    shape = coef.shape
    n = coef.size
    strides = [int(np.prod(shape[ax + 1:])) for ax in range(coef.ndim)]
    idx = np.arange(n).reshape(shape)
    diag = np.zeros(shape)
    # (offset, row-index, col-index, weight) per face orientation; lower
    # neighbours (negative offsets) first so columns come out sorted
    lower, upper = [], []
    for ax in range(coef.ndim):
        lo = [slice(None)] * coef.ndim
        hi = [slice(None)] * coef.ndim
        lo[ax] = slice(0, shape[ax] - 1)
        hi[ax] = slice(1, shape[ax])
        w = harmonic_face(coef[tuple(lo)], coef[tuple(hi)])
        diag[tuple(lo)] += w
        diag[tuple(hi)] += w
        upper.append((strides[ax], idx[tuple(lo)].ravel(), -w.ravel()))
        lower.append((-strides[ax], idx[tuple(hi)].ravel(), -w.ravel()))
        first = [slice(None)] * coef.ndim
        last = [slice(None)] * coef.ndim
        first[ax] = slice(0, 1)
        last[ax] = slice(shape[ax] - 1, shape[ax])
        diag[tuple(first)] += coef[tuple(first)]
        diag[tuple(last)] += coef[tuple(last)]
    rows, cols, vals = [], [], []
    for off, r, w in lower + upper:
        rows.append(r)
        cols.append(r + off)
        vals.append(w)
    rows.append(np.arange(n))
    cols.append(np.arange(n))
    vals.append(diag.ravel())
    return from_coo(n, np.concatenate(rows), np.concatenate(cols),
                    np.concatenate(vals))


def log_uniform_block_field(shape, block, decades, rng):
    """Piecewise-constant field: one value 10**U(-decades, decades) per
    block of ``block`` cells per axis (C3: 16x16 blocks of 32^2 cells,
    C4: 8^3 blocks of 8^3 cells)."""
    nb = tuple(s // block for s in shape)
    if any(b * block != s for b, s in zip(nb, shape)):
        raise DimensionMismatch("grid must be a multiple of the block size")
    logs = rng.uniform(-decades, decades, size=nb)
    a = 10.0 ** logs
    for ax in range(len(shape)):
        a = np.repeat(a, block, axis=ax)
    return a


def _q1_element_stiffness(h, nu):
    """24 x 24 stiffness of a cube Q1 hexahedron of side h, E = 1, 2x2x2
    Gauss points; dof order (node, component), local nodes lexicographic in
    (x, y, z) with x fastest.  Exactly symmetric."""
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    d = np.zeros((6, 6))
    d[:3, :3] = lam
    d[np.arange(3), np.arange(3)] += 2.0 * mu
    d[np.arange(3, 6), np.arange(3, 6)] = mu
    corners = np.array([[a, b, c] for c in (0, 1) for b in (0, 1) for a in (0, 1)],
                       dtype=np.float64) * 2.0 - 1.0
    g = 1.0 / np.sqrt(3.0)
    ke = np.zeros((24, 24))
    for gz in (-g, g):
        for gy in (-g, g):
            for gx in (-g, g):
                xi = np.array([gx, gy, gz])
                # dN/dxi for the 8 nodes, then dN/dx = dN/dxi * 2 / h
                dn = np.empty((8, 3))
                for a in range(8):
                    s = corners[a]
                    f = 1.0 + s * xi
                    dn[a, 0] = s[0] * f[1] * f[2] / 8.0
                    dn[a, 1] = f[0] * s[1] * f[2] / 8.0
                    dn[a, 2] = f[0] * f[1] * s[2] / 8.0
                dn *= 2.0 / h
                bm = np.zeros((6, 24))
                for a in range(8):
                    x, y, z = dn[a]
                    c = 3 * a
                    bm[0, c], bm[1, c + 1], bm[2, c + 2] = x, y, z
                    bm[3, c], bm[3, c + 1] = y, x
                    bm[4, c + 1], bm[4, c + 2] = z, y
                    bm[5, c], bm[5, c + 2] = z, x
                ke += bm.T @ d @ bm * (h ** 3 / 8.0)
    return 0.5 * (ke + ke.T)


def elasticity_q1(ne, block, decades, rng, nu=0.3):
    """3D linear elasticity on ne^3 trilinear (Q1) hexahedra of the unit
    cube, 3 dofs per node, clamped on the x = 0 face (BASELINE config C5).
    Young's modulus is piecewise constant on block^3 elements, one value
    10**U(-decades, decades) per block drawn from ``rng`` (drawn first).

    Free nodes are numbered lexicographically (x fastest) over the
    (ne+1)^3 grid minus the x = 0 face; dof = 3 * node + component.
    Returns (A, coords[n_nodes, 3])."""
    nb = ne // block
    if nb * block != ne:
        raise DimensionMismatch("element grid must be a multiple of the block size")
    young = 10.0 ** rng.uniform(-decades, decades, size=(nb, nb, nb))
    h = 1.0 / ne
    ke = _q1_element_stiffness(h, nu)
    nn = ne + 1
    gid = np.arange(nn ** 3).reshape(nn, nn, nn)       # [z, y, x]
    free = gid[:, :, 1:].ravel()
    node_of = np.full(nn ** 3, -1, dtype=np.int64)
    node_of[free] = np.arange(free.size)
    ez, ey, ex = np.meshgrid(np.arange(ne), np.arange(ne), np.arange(ne), indexing="ij")
    ez, ey, ex = ez.ravel(), ey.ravel(), ex.ravel()
    loc = [(a, b, c) for c in (0, 1) for b in (0, 1) for a in (0, 1)]
    enodes = np.stack([gid[ez + c, ey + b, ex + a] for a, b, c in loc], axis=1)
    edofs = (3 * node_of[enodes][:, :, None] + np.arange(3)).reshape(-1, 24)
    scale = young[ez // block, ey // block, ex // block]
    rows = np.repeat(edofs, 24, axis=1).ravel()
    cols = np.tile(edofs, (1, 24)).ravel()
    vals = (scale[:, None, None] * ke[None]).ravel()
    keep = (rows >= 0) & (cols >= 0)      # clamped dofs: homogeneous Dirichlet
    import scipy.sparse as sps
    n = 3 * free.size
    m = sps.coo_matrix((vals[keep], (rows[keep], cols[keep])), shape=(n, n)).tocsr()
    m.sum_duplicates()
    # duplicate sums may round differently in the two triangles: average them
    # (x + y == y + x in IEEE, so the result is exactly symmetric)
    m = ((m + m.T) * 0.5).tocsr()
    m.sort_indices()
    zz, yy, xx = np.unravel_index(free, (nn, nn, nn))
    coords = np.stack([xx, yy, zz], axis=1).astype(np.float64) * h
    a = SparseSymMatrix(n, m.indptr.astype(np.int64), m.indices.astype(np.int64),
                        m.data.astype(np.float64))
    return a, coords


def rigid_body_modes(coords, center=None):
    """The 6 rigid-body modes (3 translations, 3 rotations about ``center``,
    default the centroid of the full mesh) as an (3 n_nodes) x 6 array in the
    node-major dof order of ``elasticity_q1``."""
    c = np.full(3, 0.5) if center is None else np.asarray(center, dtype=np.float64)
    x, y, z = (coords - c).T
    nn = coords.shape[0]
    r = np.zeros((nn, 3, 6))
    for k in range(3):
        r[:, k, k] = 1.0
    r[:, 1, 3], r[:, 2, 3] = -z, y          # about x
    r[:, 0, 4], r[:, 2, 4] = z, -x          # about y
    r[:, 0, 5], r[:, 1, 5] = -y, x          # about z
    return r.reshape(3 * nn, 6)


BASELINE_CONFIGS = {
    # name: (grid, block, decades, seed, levels)
    "C1": ((128, 128), None, 0.0, 0, 7),
    "C2": ((32, 32, 32), None, 0.0, 1, 10),
    "C3": ((512, 512), 32, 3.0, 2, 12),
    "C4": ((64, 64, 64), 8, 3.0, 3, 15),
}


def baseline_problem(name, grid=None, device=False):
    """(A, b, levels) for BASELINE.json config ``name`` (C1-C5).

    C5 (elasticity) levels refer to the NODE graph (``build_hierarchy(a,
    levels, block=3)``); ``c5_problem`` also returns the coordinates.

    ``grid`` overrides the grid side (same construction, smaller size) for
    tests; the field is drawn first, then ``b = rng.standard_normal(n)``.
    ``device=True`` builds the C2-C4 matrices on the B200 (same values).
    """
    if name == "C5":
        a, b, levels, _ = c5_problem(grid)
        return a, b, levels
    shape, block, decades, seed, levels = BASELINE_CONFIGS[name]
    if grid is not None:
        shape = tuple([grid] * len(shape))
    rng = np.random.default_rng(seed)
    if block is None:
        a = (diffusion_fv_device(np.ones(shape), 1, shape) if device
             else diffusion_fv(np.ones(shape)))
    else:
        if grid is not None:
            block = max(1, min(block, grid // 8 if grid >= 8 else 1))
        if device:
            nb = tuple(s_ // block for s_ in shape)
            a = diffusion_fv_device(10.0 ** rng.uniform(-decades, decades, size=nb),
                                    block, shape)
        else:
            a = diffusion_fv(log_uniform_block_field(shape, block, decades, rng))
    b = rng.standard_normal(a.n)
    return a, b, levels


def c5_problem(ne=None):
    """BASELINE config C5: (A, b, levels, coords); ne elements per axis
    (default 24), E blocks of 4^3 elements (ne // 6 for smaller ne), seed 4,
    levels = default_levels(number of nodes) on the node graph."""
    from .partition import default_levels
    ne = 24 if ne is None else int(ne)
    block = 4 if ne == 24 else max(1, ne // 6)
    rng = np.random.default_rng(4)
    a, coords = elasticity_q1(ne, block, 2.0, rng)
    b = rng.standard_normal(a.n)
    return a, b, default_levels(coords.shape[0]), coords
