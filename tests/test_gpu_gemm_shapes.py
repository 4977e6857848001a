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
