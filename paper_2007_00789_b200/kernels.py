"""Thin Python wrappers over the batched C-ABI kernels.

``Geometry`` holds the device ``m0``/``off`` arrays that every batched
factorization kernel reads (see include/spand_b200.h): real clusters plus
"virtual" clusters for workspaces and one-off matrices.  ``*_one`` helpers
run a single task (the reference's per-block dense API in ``dense.py``).
"""

import numpy as np

from . import _lib
from .device import dev, ptr, require_cuda, stream, to_dev, to_dev_async


def opnd(p, rc, cc, rskip=0, cskip=0, rcount=-1, ccount=-1):
    """Operand row (7 int64): see include/spand_b200.h."""
    return [int(p), int(rc), int(cc), int(rskip), int(cskip), int(rcount),
            int(ccount)]


class Geometry:
    """Device geometry table (int32 m0 and off)."""

    def __init__(self, m0, off=None):
        t = require_cuda()
        m0 = np.asarray(m0, dtype=np.int32)
        self.m0_host = m0.copy()
        self.m0 = to_dev(m0, np.int32)
        self.off = (to_dev(np.asarray(off, np.int32), np.int32) if off is not None
                    else t.zeros(m0.size, dtype=t.int32, device=dev()))

    @classmethod
    def virtual(cls, sizes):
        return cls(np.asarray(sizes, dtype=np.int32))


def _rows(rows, width):
    return to_dev_async(np.asarray(rows, dtype=np.int64).reshape(-1, width))


def potrf_batched(geo, ops, info):
    n = len(ops)
    if n == 0:
        return
    d = _rows([list(o) + [i] for i, o in enumerate(ops)], 8)
    _lib.call("spand_potrf_batched", n, ptr(d), ptr(geo.m0), ptr(geo.off),
              ptr(info), 0, 0, stream())


def trtri_batched(geo, pairs, sizes=None):
    """Lower-triangular inverses X = L^-1 for [(L operand, X operand)].

    ``sizes`` (max live size per pair, default the m0 of the row cluster)
    drive the recursive doubling: 64x64 diagonal tiles are inverted in
    shared memory, then level r combines 2^r-tile blocks with two grouped
    DMMA GEMMs, T = B A^-1 and X_21 = -C^-1 T."""
    n = len(pairs)
    if n == 0:
        return
    if sizes is None:
        sizes = [int(geo.m0_host[l[1]]) for l, _ in pairs]
    t = require_cuda()
    tiles = []
    for (l, x), nm in zip(pairs, sizes):
        for o in range(0, nm, TILE):
            tiles.append(_sub(l, o, o, TILE, TILE) + _sub(x, o, o, TILE, TILE))
    if tiles:
        d = _rows(tiles, 14)
        _lib.call("spand_trtri_tiles", len(tiles), ptr(d), ptr(geo.m0),
                  ptr(geo.off), stream())
    nmax = max(sizes) if sizes else 0
    if nmax <= TILE:
        return
    # temp with the same geometry as each X (m0^2 of the row cluster)
    toff, acc = [], 0
    for l, _ in pairs:
        toff.append(acc)
        acc += int(geo.m0_host[l[1]]) ** 2
    temp = t.empty(max(acc, 1), dtype=t.float64, device=dev())
    tb = temp.data_ptr()
    s = TILE
    while s < nmax:
        g1, g2 = [], []
        for (l, x), nm, to in zip(pairs, sizes, toff):
            tmp = [tb + 8 * to] + x[1:]
            for o in range(0, nm - s, 2 * s):
                # T = B A^-1 with B = L[o+s:o+2s, o:o+s], A^-1 = X[o:o+s, o:o+s]
                g1.append((_sub(tmp, o + s, o, s, s),
                           [(_sub(l, o + s, o, s, s), _sub(x, o, o, s, s))],
                           (s, s)))
                # X[o+s:o+2s, o:o+s] = -C^-1 T
                g2.append((_sub(x, o + s, o, s, s),
                           [(_sub(x, o + s, o + s, s, s), _sub(tmp, o + s, o, s, s))],
                           (s, s)))
        gemm_grouped(geo, g1, 1.0, 0.0, bT=0, tri=4)
        gemm_grouped(geo, g2, -1.0, 0.0, bT=0, tri=1)
        s *= 2
    # `temp` may be released now: the caching allocator hands the block to
    # later allocations on this stream only, i.e. after these GEMMs


def _sub(o, rskip, cskip, rcount, ccount):
    """Sub-operand of an operand row (skips are relative to its start)."""
    return [o[0], o[1], o[2], o[3] + rskip, o[4] + cskip,
            rcount if o[5] < 0 else min(rcount, max(o[5] - rskip, 0)),
            ccount if o[6] < 0 else min(ccount, max(o[6] - cskip, 0))]


def copy_batched(geo, tasks):
    """tasks: [(src operand, dst operand, mode)]"""
    n = len(tasks)
    if n == 0:
        return
    d = _rows([a + b + [m] for a, b, m in tasks], 15)
    _lib.call("spand_copy_batched", n, ptr(d), ptr(geo.m0), ptr(geo.off),
              stream())


TILE = 64
# grouped-GEMM tile shapes (gemm.cu, `tri >> 4`; planner.h kShapeM / kShapeN)
SHAPES = ((64, 64), (64, 16), (32, 32), (16, 16), (16, 64), (64, 32), (32, 64))


def _tile_grid(mm, nn, lower_only=False, shape=0):
    """All (target, i0, j0) tiles of targets with extents mm x nn."""
    TM, TN = SHAPES[shape]
    tm = np.maximum(-(-mm // TM), 0)
    tn = np.maximum(-(-nn // TN), 0)
    cnt = tm * tn
    tot = int(cnt.sum())
    if tot == 0:
        return np.zeros(0, dtype=np.int64)
    tgt = np.repeat(np.arange(mm.size, dtype=np.int64), cnt)
    local = np.arange(tot, dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    ntile_n = np.repeat(tn, cnt)
    i0 = (local // ntile_n) * TM
    j0 = (local % ntile_n) * TN
    out = (tgt << 32) | ((i0 // TM) << 16) | (j0 // TN)
    if lower_only:
        out = out[j0 < i0 + TM]
    return out


def gemm_grouped(geo, targets, alpha, beta, bT, lower_only=False,
                 max_rows=None, max_cols=None, tri=0, shape=0, mask_rows=None):
    """targets: [(C operand, [(A operand, B operand), ...], (max_m, max_n))].

    Tiles are laid out for the maximal (m0-geometry) sizes; tiles beyond a
    target's live size exit immediately on the device.

    ``mask_rows`` (one segment per target): the row counts of the masked
    operand -- B for bT = 0 (its zero 16-row K chunks are skipped), A for
    bT = 1 (tiles over zero rows of A write zeros at once).  The masks are
    written by ``spand_gemm_kmask`` and the product runs through
    ``spand_gemm_grouped_masked`` (bit-identical to the unmasked call)."""
    if not targets:
        return
    trow, srow = [], []
    mm = np.empty(len(targets), dtype=np.int64)
    nn = np.empty(len(targets), dtype=np.int64)
    for t, (c, segs, (mt, nt)) in enumerate(targets):
        trow.append(c + [len(srow)])
        for a, b in segs:
            srow.append(a + b)
        mm[t], nn[t] = mt, nt
    trow.append([0] * 7 + [len(srow)])
    tiles = _tile_grid(mm, nn, lower_only, shape)
    if tiles.shape[0] == 0:
        return
    if not srow:
        srow.append([0] * 14)
    td, sd, tl = _rows(trow, 8), _rows(srow, 14), _rows(tiles, 1)
    if mask_rows is not None:
        t = require_cuda()
        chunks = (np.asarray(mask_rows, dtype=np.int64) + 15) // 16
        kmoff = np.concatenate([[0], np.cumsum(chunks)[:-1]]).astype(np.int64)
        kd = _rows(kmoff, 1)
        mask = t.full((int(chunks.sum()) + 1,), 255, dtype=t.uint8, device=dev())
        _lib.call("spand_gemm_kmask", len(targets), ptr(td), ptr(sd), ptr(geo.m0),
                  ptr(geo.off), ptr(mask), ptr(kd), 0 if bT else 1, stream())
        _lib.call("spand_gemm_grouped_masked", int(tiles.shape[0]), ptr(tl), ptr(td), ptr(sd),
                  ptr(geo.m0), ptr(geo.off), float(alpha), float(beta), int(bT),
                  int(bool(lower_only)), int(tri) | (int(shape) << 4), None, 0,
                  ptr(mask), ptr(kd), stream())
        return mask
    _lib.call("spand_gemm_grouped", int(tiles.shape[0]), ptr(tl), ptr(td), ptr(sd),
              ptr(geo.m0), ptr(geo.off), float(alpha), float(beta), int(bT),
              int(bool(lower_only)), int(tri) | (int(shape) << 4), None, 0, stream())


# ---------------------------------------------------------------------------
# single-task helpers for the reference's dense API


def _colmajor_upload(a):
    return to_dev(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T).ravel())


def _download(buf, rows, cols):
    return buf[:rows * cols].cpu().numpy().reshape(cols, rows).T.copy()


def potrf_one(a):
    t = require_cuda()
    n = a.shape[0]
    geo = Geometry.virtual([n])
    buf = _colmajor_upload(a)
    info = t.zeros(1, dtype=t.int32, device=dev())
    potrf_batched(geo, [opnd(buf.data_ptr(), 0, 0)], info)
    return _download(buf, n, n), int(info.item())


def trtri_one(l):
    t = require_cuda()
    n = l.shape[0]
    geo = Geometry.virtual([n])
    src = _colmajor_upload(l)
    dst = t.zeros(n * n, dtype=t.float64, device=dev())
    trtri_batched(geo, [(opnd(src.data_ptr(), 0, 0), opnd(dst.data_ptr(), 0, 0))])
    return _download(dst, n, n)


def gemm_one(a, b, trans_a=False, trans_b=False):
    """C = op(A) op(B) on the DMMA GEMM (A, B host arrays)."""
    t = require_cuda()
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if trans_a:
        a = a.T
    m, k = a.shape
    k2, nn = (b.shape[1], b.shape[0]) if trans_b else b.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    geo = Geometry.virtual([m, k, nn])
    ad = _colmajor_upload(a)                     # m x k
    if trans_b:
        bd = _colmajor_upload(b)                 # n x k  ("NT")
        bop = opnd(bd.data_ptr(), 2, 1)
        bT = 1
    else:
        bd = _colmajor_upload(b)                 # k x n  ("NN")
        bop = opnd(bd.data_ptr(), 1, 2)
        bT = 0
    cd = t.zeros(max(m * nn, 1), dtype=t.float64, device=dev())
    gemm_grouped(geo, [(opnd(cd.data_ptr(), 0, 2),
                        [(opnd(ad.data_ptr(), 0, 1), bop)], (m, nn))],
                 1.0, 0.0, bT)
    return _download(cd, m, nn)


def rrqr_one(a, eps, scheme):
    from .rrqr import rrqr_single
    return rrqr_single(a, eps, scheme)
