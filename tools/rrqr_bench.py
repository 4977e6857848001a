"""Time the RRQR wave kernel on one large synthetic panel (GPU-generated)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2007_00789_b200 import _lib
from paper_2007_00789_b200.device import dev, ptr, stream, to_dev
from paper_2007_00789_b200.kernels import Geometry
m, n, rank = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
G = int(sys.argv[4]) if len(sys.argv) > 4 else _lib.load().spand_rrqr_capacity(m)
torch.manual_seed(0)
# A = U diag(s) V^T with geometric singular values: rank ~ `rank` above 1e-2
s = torch.logspace(0, -4 * min(m, n) / rank, min(m, n), dtype=torch.float64, device="cuda")
U = torch.linalg.qr(torch.randn(m, min(m, n), dtype=torch.float64, device="cuda"))[0]
Vt = torch.randn(min(m, n), n, dtype=torch.float64, device="cuda") / n ** 0.5
A = (U * s) @ Vt
blk = A.t().contiguous().reshape(-1)   # column-major m x n
geo = Geometry(np.array([m, n], dtype=np.int32))
ncap, mcap = n, m
wsz = mcap * ncap + mcap * mcap + 32 * (ncap + mcap)
asz = 2 * ncap + 3 * mcap + 68 * G + 8
isz = (3 * ncap + 1) // 2 + 1
work = torch.zeros(wsz + asz + isz + 1, dtype=torch.float64, device="cuda")
q = torch.zeros(m * m, dtype=torch.float64, device="cuda")
ev = torch.zeros(12, dtype=torch.int64, device="cuda")
times = []
ev.zero_()
for rep in range(3):
    b2 = blk.clone()
    ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
    wb = work.data_ptr()
    prow = [[0, 0, 1, wb, q.data_ptr(), wb + 8 * wsz, wb + 8 * (wsz + asz), 0, G, ctr.data_ptr(), 0, ncap, mcap, 0, 0, 0]]
    nrow = [[1, b2.data_ptr(), 0, 0]]
    pd, nd = to_dev(np.asarray(prow, np.int64)), to_dev(np.asarray(nrow, np.int64))
    geo.off.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("spand_rrqr_wave", 1, G, m, ptr(pd), ptr(nd), ptr(geo.m0), ptr(geo.off), 1e-2, 1, ptr(ev), stream())
    e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
e = ev.cpu().numpy()
k = int(e[3])
ks = np.arange(k, dtype=np.float64)
traffic = float(np.sum(8.0 * (m - ks) * (n - ks)))   # one read of the trailing panel per step
print(json.dumps({"stale_recomputes": int(e[10]) // 3, "m": m, "n": n, "G": G, "k_stop": k, "k_c": int(e[4]), "ms": times, "ms_per_step": min(times) / max(k, 1),
                  "GBs_1read_per_step": traffic / (min(times) / 1e3) / 1e9}))
