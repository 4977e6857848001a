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
bad = 0
for (m, n) in [(20, 40), (64, 200), (128, 300), (200, 900)]:
    sv = np.geomspace(1, 1e-6, min(m, n))
    a = wsv(m, n, sv, m)
    for scheme in ("first", "second-full", "second-superfine"):
        ref = orc.sparsify_panel(a, 1e-2, scheme)
        for g in (1, 3, 40):
            r = rrqr_single(a, 1e-2, scheme, group=g)
            ok = r.rank_c == ref["rank_c"] and r.rank_f2 == ref["rank_f2"]
            err = np.abs(r.r_coarse - ref["r_coarse"]).max() / np.abs(ref["r_coarse"]).max() if ok and r.rank_c else 0
            eerr = np.abs(r.e_tilde - ref["e_tilde"]).max() / max(np.abs(ref["e_tilde"]).max(), 1e-300) if ok and r.e_tilde.size else 0
            qerr = np.abs(np.hstack([r.q_c, r.q_f]) - np.hstack([ref["q_c"], ref["q_f"]])).max() if ok else None
            flag = "" if ok and err < 1e-10 and eerr < 1e-8 and qerr < 1e-10 else "  <-- BAD"
            bad += bool(flag)
            print(m, n, scheme, g, "rank", r.rank_c, ref["rank_c"], r.rank_f2, ref["rank_f2"], "rerr %.1e eerr %.1e qerr %s" % (err, eerr, qerr), flag, flush=True)
print("bad", bad)
