import sys, numpy as np
sys.path.insert(0, '.')
from oracle import spand_oracle as orc
from paper_2007_00789_b200.rrqr import rrqr_single
rng = np.random.default_rng(0)
bad = 0
for (m, n) in [(8, 16), (40, 100), (100, 500), (300, 2000), (70, 40)]:
    a = rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, n)))
    for eps in (1e-2, 1e-8):
        ref = orc.sparsify_panel(a, eps, "second-full")
        for g in (1, 7, 50, 200):
            r = rrqr_single(a, eps, "second-full", group=g)
            ok = r.rank_c == ref["rank_c"]
            err = np.abs(r.r_coarse - ref["r_coarse"]).max() / np.abs(ref["r_coarse"]).max() if ok and r.rank_c else 0
            eerr = np.abs(r.e_tilde - ref["e_tilde"]).max() / max(np.abs(ref["e_tilde"]).max(), 1e-300) if ok and r.e_tilde.size else 0
            qerr = np.abs(np.hstack([r.q_c, r.q_f]) - np.hstack([ref["q_c"], ref["q_f"]])).max() if ok else None
            flag = "" if ok and err < 1e-10 and eerr < 1e-8 and qerr < 1e-10 else "  <-- BAD"
            bad += bool(flag)
            print(m, n, eps, g, "rank", r.rank_c, ref["rank_c"], "rerr %.1e eerr %.1e qerr %s" % (err, eerr, qerr), flag, flush=True)
print("bad", bad)
