"""Single-panel entry to the RRQR wave kernel (reference `rrqr_sparsify`).

The factorization launches whole waves of interfaces at once from
``engine.py``; this module drives the same kernel for one stand-alone panel
(``dense.rrqr_sparsify``), using a two-cluster geometry: cluster 0 is the
panel's row set, cluster 1 its column set, and the panel is block (0, 1).
"""

import numpy as np

from . import _lib
from .dense import SCHEME_CODE, RRQRResult, SchemeKind
from .device import dev, ptr, require_cuda, stream, to_dev
from .kernels import Geometry

MAX_ROWS = 24576   # rrqr.cu kMaxM


def rrqr_single(a, eps, scheme, group=None, pad=0, cluster=0):
    """``pad`` > 0 stores the panel inside a larger block (live window at an
    offset, as for an interface sparsified for the second time).
    ``cluster`` = 2, 4 or 8 runs the clustered variant of the kernel
    (``spand_rrqr_wave_clustered``) with ``group`` CTAs (a multiple of it)."""
    t = require_cuda()
    m, n = a.shape
    if m > MAX_ROWS:
        from .errors import PanelTooLarge
        raise PanelTooLarge(m, MAX_ROWS)
    mp, np_ = m + pad, n + pad
    geo = Geometry(np.array([mp, np_], dtype=np.int32),
                   np.array([pad, pad], dtype=np.int32))
    big = np.zeros((mp, np_))
    big[pad:, pad:] = a
    blk = to_dev(np.ascontiguousarray(big.T).ravel() if big.size else np.zeros(1))
    cap = max(1, _lib.load().spand_rrqr_capacity(max(m, 1)))
    g = group or max(1, min(cap, n // 64, (m * n) // 65536 + 1))
    if cluster > 1:
        # co-resident clusters bound the group (cooperative launch)
        ccap = _lib.load().spand_rrqr_cluster_capacity(max(m, 1), cluster)
        if ccap >= cluster:
            g = min(g, ccap)
        g = max(cluster, (g // cluster) * cluster)
    ncap, mcap = max(np_, 1), max(mp, 1)
    wsz = mcap * ncap + mcap * mcap + 32 * (ncap + mcap) + 32 * mcap + 1024   # + T blocks
    asz = 2 * ncap + 3 * mcap + 2 * g * 34 + 8 + 1024
    isz = (3 * ncap + 1) // 2 + 1
    work = t.zeros(wsz + asz + isz + 1, dtype=t.float64, device=dev())
    q = t.zeros(mcap * mcap, dtype=t.float64, device=dev())
    ctr = t.zeros(2, dtype=t.int32, device=dev())
    events = t.zeros(12, dtype=t.int64, device=dev())
    wb = work.data_ptr()
    lists = None
    if cluster > 1:
        lists = t.zeros(4 * g * (ncap // (g // cluster) + 2) + 2, dtype=t.int32, device=dev())
    prow = [[0, 0, 1, wb, q.data_ptr(), wb + 8 * wsz, wb + 8 * (wsz + asz), 0, g,
             ctr.data_ptr(), 0, ncap, mcap, 0,
             lists.data_ptr() if lists is not None else 0, 0]]
    nrow = [[1, blk.data_ptr(), 0, 0]]
    pd = to_dev(np.asarray(prow, dtype=np.int64))
    nd = to_dev(np.asarray(nrow, dtype=np.int64))
    if isinstance(scheme, str):
        scheme = SchemeKind.from_string(scheme)
    if cluster > 1:
        _lib.call("spand_rrqr_wave_clustered", 1, g, max(m, 1), cluster, ptr(pd), ptr(nd),
                  ptr(geo.m0), ptr(geo.off), float(eps), SCHEME_CODE[scheme], ptr(events),
                  stream())
    else:
        _lib.call("spand_rrqr_wave", 1, g, max(m, 1), ptr(pd), ptr(nd), ptr(geo.m0),
                  ptr(geo.off), float(eps), SCHEME_CODE[scheme], ptr(events), stream())
    ev = events.cpu().numpy()
    k_stop, k_c, n_fine = int(ev[3]), int(ev[4]), int(ev[6])
    qh = q[:m * m].cpu().numpy().reshape(m, m).T.copy() if m else np.zeros((0, 0))
    bh = (blk[:mp * np_].cpu().numpy().reshape(np_, mp).T[pad:, pad:].copy()
          if m * n else np.zeros((m, n)))
    iaux = work[wsz + asz:wsz + asz + isz].cpu().numpy().view(np.int32)
    perm = iaux[:n].astype(np.int64)
    r_coarse = np.ascontiguousarray(bh[n_fine:, :]) if k_c else np.zeros((0, n))
    if scheme is SchemeKind.FIRST_ORDER:
        e_tilde, rank_f2 = np.zeros((0, n)), 0
    elif scheme is SchemeKind.SECOND_ORDER_FULL:
        e_tilde, rank_f2 = np.ascontiguousarray(bh[:n_fine, :]), 0
    else:
        rank_f2 = k_stop - k_c
        e_tilde = np.ascontiguousarray(bh[:rank_f2, :])
    if n == 0:
        perm = np.arange(0)
    return RRQRResult(perm=perm, q_c=np.ascontiguousarray(qh[:, :k_c]),
                      q_f=np.ascontiguousarray(qh[:, k_c:]), r_coarse=r_coarse,
                      e_tilde=e_tilde, rank_c=k_c, rank_f2=rank_f2)
