"""Several independent panels in ONE cooperative RRQR launch (engine-like)."""
import sys, numpy as np
sys.path.insert(0, '.')
import torch
from oracle import spand_oracle as orc
from paper_2007_00789_b200 import _lib
from paper_2007_00789_b200.device import dev, ptr, stream, to_dev
from paper_2007_00789_b200.kernels import Geometry

def wsv(m, n, sv, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.zeros((m, n)); k = min(len(sv), m, n); s[:k, :k] = np.diag(sv[:k])
    return u @ s @ v.T

def run(panels, groups, eps, code, fill):
    P = len(panels)
    m0 = []
    for a in panels:
        m0 += [a.shape[0], a.shape[1]]
    geo = Geometry(np.array(m0, dtype=np.int32))
    blks = [to_dev(np.ascontiguousarray(a.T).ravel()) for a in panels]
    cap = _lib.load().spand_rrqr_cta_count()
    assert sum(groups) <= cap, (sum(groups), cap)
    lay, need = [], 0
    for a, g in zip(panels, groups):
        m, n = a.shape
        wsz = m * n + m * m + 32 * (n + m); asz = 2 * n + 3 * m + 68 * g + 8; isz = (3 * n + 1) // 2 + 1
        lay.append((need, wsz, asz, isz)); need += wsz + asz + isz + 1
    work = torch.full((need,), fill, dtype=torch.float64, device=dev())
    qs = [torch.zeros(a.shape[0] ** 2, dtype=torch.float64, device=dev()) for a in panels]
    ctr = torch.zeros(P, dtype=torch.int32, device=dev())
    ev = torch.zeros(12 * P, dtype=torch.int64, device=dev())
    wb = work.data_ptr()
    prow, nrow, gb = [], [], 0
    for i, (a, g, (at, wsz, asz, isz)) in enumerate(zip(panels, groups, lay)):
        m, n = a.shape
        nrow.append([2 * i + 1, blks[i].data_ptr(), 0, 0])
        prow.append([2 * i, i, i + 1, wb + 8 * at, qs[i].data_ptr(), wb + 8 * (at + wsz), wb + 8 * (at + wsz + asz),
                     gb, g, ctr.data_ptr() + 4 * i, i, n, m, 0, 0, 0])
        gb += g
    pd = to_dev(np.asarray(prow, dtype=np.int64)); nd = to_dev(np.asarray(nrow, dtype=np.int64))
    _lib.call("spand_rrqr_wave", P, gb, max(a.shape[0] for a in panels), ptr(pd), ptr(nd), ptr(geo.m0), ptr(geo.off),
              float(eps), code, ptr(ev), stream())
    torch.cuda.synchronize()
    return ev.cpu().numpy().reshape(P, 12), [b.cpu().numpy() for b in blks]

bad = 0
rng = np.random.default_rng(5)
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    P = int(rng.integers(1, 5))
    panels = []
    for i in range(P):
        m = int(rng.integers(3, 40)); n = int(rng.integers(3, 60))
        panels.append(wsv(m, n, np.geomspace(1, 1e-5, min(m, n)), int(rng.integers(1000))))
    groups = [int(rng.integers(1, 120)) for _ in range(P)]
    fill = float(rng.choice([0.0, np.nan, 1e300]))
    ev, blks = run(panels, groups, 0.05, 0, fill)
    for i, a in enumerate(panels):
        ref = orc.sparsify_panel(a, 0.05, "first")
        m, n = a.shape
        b = blks[i].reshape(n, m).T
        nf = m - ref["rank_c"]
        ok = ev[i, 4] == ref["rank_c"] and np.allclose(b[nf:, :], ref["r_coarse"], atol=1e-10)
        if not ok:
            bad += 1
            print("trial", trial, "panel", i, (m, n), "G", groups[i], "fill", fill, "k_c", ev[i, 4], ref["rank_c"], flush=True)
print("bad", bad, flush=True)
