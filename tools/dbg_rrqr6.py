import sys, numpy as np
sys.path.insert(0, '.')
from oracle import spand_oracle as orc
from paper_2007_00789_b200.rrqr import rrqr_single
def wsv(m, n, sv, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.zeros((m, n)); k = min(len(sv), m, n); s[:k, :k] = np.diag(sv[:k])
    return u @ s @ v.T
for (m, n) in [(8, 10), (20, 40), (64, 200)]:
    a = wsv(m, n, np.geomspace(1, 1e-6, min(m, n)), m)
    ref = orc.sparsify_panel(a, 1e-2, "second-full")
    for pad in (0, 3, 8):
        r = rrqr_single(a, 1e-2, "second-full", group=1, pad=pad)
        print(m, n, pad, "rank", r.rank_c, ref["rank_c"], "rc err %.2e" % np.abs(r.r_coarse - ref["r_coarse"]).max(), "e err %.2e" % np.abs(r.e_tilde - ref["e_tilde"]).max(), flush=True)
