"""Every tile shape of the grouped DMMA GEMM (gemm.cu; the planner picks one
per target, planner.h tile_shape) against NumPy on mixed target sizes: NN and
NT, several K-concatenated segments per target, triangular K bounds
(tri 1 / 2 / 4) and lower-only diagonal targets."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12   # relative Frobenius; FP64 products of O(1) entries, K <= 200


def _run(shape, bT, tri, lower_only, seed):
    import torch
    from paper_2007_00789_b200 import kernels as K
    from paper_2007_00789_b200.device import dev
    rng = np.random.default_rng(seed)
    sizes = [(3, 5), (6, 6), (17, 9), (40, 13), (70, 30), (129, 65), (16, 70)]
    bufs, targets, ref = [], [], []
    m0 = []

    def upload(a):
        d = torch.from_numpy(np.ascontiguousarray(a.T).ravel().copy()).to(dev())
        bufs.append(d)
        return d.data_ptr()

    def cluster(n):
        m0.append(n)
        return len(m0) - 1

    for (m, n) in sizes:
        if lower_only:
            n = m
        segs, acc = [], np.zeros((m, n))
        for _ in range(2):
            k = m if tri & 1 else (n if tri & 6 else int(rng.integers(1, 40)))
            a = rng.standard_normal((m, k))
            if tri & 1:
                a = np.tril(a)
            b = rng.standard_normal((n, k) if bT else (k, n))
            if tri & 2:
                b = np.tril(b)
            if tri & 4:
                b = np.tril(b)
            acc += a @ (b.T if bT else b)
            ca, ck, cn = cluster(m), cluster(k), cluster(n)
            bop = K.opnd(upload(b), cn, ck) if bT else K.opnd(upload(b), ck, cn)
            segs.append((K.opnd(upload(a), ca, ck), bop))
        c0 = rng.standard_normal((m, n))
        cm, cn2 = cluster(m), cluster(n)
        targets.append((K.opnd(upload(c0), cm, cn2), segs, (m, n)))
        ref.append((0.5 * c0 - 2.0 * acc, lower_only))
    geo = K.Geometry(np.asarray(m0, dtype=np.int32))
    K.gemm_grouped(geo, targets, -2.0, 0.5, bT, lower_only=lower_only, tri=tri, shape=shape)
    torch.cuda.synchronize()
    for (c, segs, (m, n)), (want, lo) in zip(targets, ref):
        got = None
        for d in bufs:
            if d.data_ptr() == c[0]:
                got = d.cpu().numpy().reshape(n, m).T
        if lo:   # only the lower triangle is defined for lower-only targets
            got, want = np.tril(got), np.tril(want)
        err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
        assert err < TOL, (shape, bT, tri, lower_only, m, n, err)


@pytest.mark.parametrize("shape", range(7))
@pytest.mark.parametrize("bT,tri", [(0, 0), (1, 0), (0, 1), (1, 2), (0, 4)])
def test_gemm_shape(shape, bT, tri):
    _run(shape, bT, tri, False, seed=10 * shape + tri + bT)


@pytest.mark.parametrize("shape", range(7))
def test_gemm_shape_lower_only(shape):
    _run(shape, 1, 0, True, seed=100 + shape)


def _row_sparse(rng, rows, cols, keep):
    a = np.zeros((rows, cols))
    idx = rng.choice(rows, size=max(1, int(keep * rows)), replace=False)
    a[idx] = rng.standard_normal((idx.size, cols))
    return a


@pytest.mark.parametrize("shape", range(7))
@pytest.mark.parametrize("bT", [0, 1])
def test_masked_gemm_is_bitwise_the_dense_product(shape, bT):
    """Row-chunk masks (spand_gemm_kmask + spand_gemm_grouped_masked): bT = 0
    is the interface rescale Z^-1 B (A lower triangular, B with few nonzero
    rows: its zero K chunks are skipped), bT = 1 the panel TRSM A L^-T (tiles
    over zero rows of A leave at once).  Same bits as the unmasked launch,
    and the masks equal the row-chunk pattern of the masked operand."""
    import torch
    from paper_2007_00789_b200 import kernels as K
    from paper_2007_00789_b200.device import dev
    rng = np.random.default_rng(500 + 10 * shape + bT)
    sizes = [(200, 7), (333, 40), (64, 64), (150, 17), (97, 130), (16, 5)]
    keep = []

    def upload(a):
        d = torch.from_numpy(np.ascontiguousarray(a.T).ravel().copy()).to(dev())
        keep.append(d)
        return d

    m0, built, pattern = [], [], []
    for (m, n) in sizes:
        if bT == 0:
            a = np.tril(rng.standard_normal((m, m)))          # Z^-1: m x m lower
            b = _row_sparse(rng, m, n, 0.08)                   # unscaled block: m x n
            k, masked = m, b
        else:
            k = n
            a = _row_sparse(rng, m, k, 0.08)                   # panel: m x k
            b = np.tril(rng.standard_normal((k, k)))           # L^-1: k x k lower, C = A B^T
            n, masked = k, a
        cm, ck, cn = len(m0), len(m0) + 1, len(m0) + 2
        m0 += [m, k, n]
        built.append((a, b, m, n, cm, ck, cn))
        pattern.append([bool(np.any(masked[16 * c:16 * c + 16])) for c in range((masked.shape[0] + 15) // 16)])
    geo = K.Geometry(np.asarray(m0, dtype=np.int32))
    outs = []
    for use_mask in (False, True):
        targets, cs = [], []
        for (a, b, m, n, cm, ck, cn) in built:
            ad, bd = upload(a), upload(b)
            cd = upload(np.full((m, n), 7.0))
            cs.append((cd, m, n))
            bop = K.opnd(bd.data_ptr(), cn, ck) if bT else K.opnd(bd.data_ptr(), ck, cn)
            targets.append((K.opnd(cd.data_ptr(), cm, cn),
                            [(K.opnd(ad.data_ptr(), cm, ck), bop)], (m, n)))
        rows = [t[2][0] for t in targets] if use_mask else None
        mask = K.gemm_grouped(geo, targets, 1.0, 0.0, bT, tri=2 if bT else 1, shape=shape,
                              mask_rows=rows)
        torch.cuda.synchronize()
        outs.append([d.cpu().numpy().reshape(n, m).T.copy() for d, m, n in cs])
        if use_mask:
            got = mask.cpu().numpy()
            at = 0
            for pat in pattern:
                assert [bool(x) for x in got[at:at + len(pat)]] == pat
                at += len(pat)
    for (a, b, m, n, *_), dense, masked_out in zip(built, *outs):
        want = a @ (b.T if bT else b)
        assert np.linalg.norm(dense - want) <= TOL * max(np.linalg.norm(want), 1.0)
        assert np.array_equal(dense, masked_out)


@pytest.mark.parametrize("shape", [0, 1, 2, 5])
def test_flagged_schur_segments_are_bitwise_the_dense_update(shape):
    """Compact (Schur) segments with the panels' row-chunk flags: a tile opens
    only the segments whose A rows and B rows hold a nonzero in its ranges,
    in their original order -- same bits as opening every segment."""
    import torch
    from paper_2007_00789_b200 import _lib, kernels as K
    from paper_2007_00789_b200.device import dev, ptr, stream
    rng = np.random.default_rng(900 + shape)
    wsz, ssz = [150, 90, 40, 70], [16, 12, 20, 8, 16, 5]
    m0 = wsz + ssz
    nw, ns = len(wsz), len(ssz)
    keep = []

    def upload(a):
        d = torch.from_numpy(np.ascontiguousarray(a.T).ravel().copy()).to(dev())
        keep.append(d)
        return d

    panels, btab, pan_rows = {}, [], []
    for w in range(nw):
        for s_ in range(ns):
            pw = _row_sparse(rng, wsz[w], ssz[s_], 0.1)
            d = upload(pw)
            panels[(w, s_)] = (pw, len(btab))
            btab.append([d.data_ptr(), w, nw + s_])
            pan_rows.append(wsz[w])
    geo = K.Geometry(np.asarray(m0, dtype=np.int32))
    # row-chunk flags of every panel: one fake target per panel, A = the panel
    chunks = (np.asarray(pan_rows, dtype=np.int64) + 15) // 16
    poff = np.concatenate([[0], np.cumsum(chunks)[:-1]]).astype(np.int64)
    ftr = [[0] * 7 + [i] for i in range(len(btab))] + [[0] * 7 + [len(btab)]]
    fsr = [K.opnd(b[0], b[1], b[2]) + [0] * 7 for b in btab]
    mask = torch.full((int(chunks.sum()) + 1,), 255, dtype=torch.uint8, device=dev())
    ftd, fsd, pod = K._rows(ftr, 8), K._rows(fsr, 14), K._rows(poff, 1)
    _lib.call("spand_gemm_kmask", len(btab), ptr(ftd), ptr(fsd), ptr(geo.m0), ptr(geo.off),
              ptr(mask), ptr(pod), 0, stream())
    pairs = [(a, b) for a in range(nw) for b in range(a, nw)]
    c0 = {pq: rng.standard_normal((wsz[pq[0]], wsz[pq[1]])) for pq in pairs}
    bt = K._rows(btab, 3)
    outs = []
    for use_flags in (False, True):
        trow, srow, sflag, cds = [], [], [], []
        for (a, b) in pairs:
            cd = upload(c0[(a, b)])
            cds.append(cd)
            trow.append(K.opnd(cd.data_ptr(), a, b) + [len(srow)])
            for s_ in range(ns):
                ia, ib = panels[(a, s_)][1], panels[(b, s_)][1]
                srow.append((ia << 32) | ib)
                sflag.append((int(poff[ia]) << 32) | int(poff[ib]))
        trow.append([0] * 7 + [len(srow)])
        mm = np.array([wsz[a] for a, _ in pairs], dtype=np.int64)
        nn = np.array([wsz[b] for _, b in pairs], dtype=np.int64)
        tiles = K._tile_grid(mm, nn, False, shape)
        td, sd, tl, fd = K._rows(trow, 8), K._rows(srow, 1), K._rows(tiles, 1), K._rows(sflag, 1)
        if use_flags:
            _lib.call("spand_gemm_grouped_masked", int(tiles.shape[0]), ptr(tl), ptr(td), ptr(sd),
                      ptr(geo.m0), ptr(geo.off), -1.0, 1.0, 1, 0, shape << 4, ptr(bt), 1,
                      ptr(mask), ptr(fd), stream())
        else:
            _lib.call("spand_gemm_grouped", int(tiles.shape[0]), ptr(tl), ptr(td), ptr(sd),
                      ptr(geo.m0), ptr(geo.off), -1.0, 1.0, 1, 0, shape << 4, ptr(bt), 1, stream())
        torch.cuda.synchronize()
        outs.append([cd.cpu().numpy().reshape(wsz[b], wsz[a]).T.copy()
                     for cd, (a, b) in zip(cds, pairs)])
    for (a, b), dense, flagged in zip(pairs, *outs):
        want = c0[(a, b)] - sum(panels[(a, s_)][0] @ panels[(b, s_)][0].T for s_ in range(ns))
        assert np.linalg.norm(dense - want) <= TOL * max(np.linalg.norm(want), 1.0)
        assert np.array_equal(dense, flagged)
