import sys, glob, numpy as np
sys.path.insert(0, '.')
from oracle import spand_oracle as orc
from paper_2007_00789_b200.rrqr import rrqr_single
for f in sorted(glob.glob("gpurun_out/bad_rc_panel_*.npy"))[:3]:
    a = np.load(f)
    for eps in (0.05,):
        ref = orc.sparsify_panel(a, eps, "second-full")
        for g in (1,):
            r = rrqr_single(a, eps, "second-full", group=g)
            print(f, a.shape, "rank", r.rank_c, ref["rank_c"], "rc err", np.abs(r.r_coarse - ref["r_coarse"]).max(), "perm", r.perm[:10], ref["perm"][:10])
            print(np.round(r.r_coarse[:3, :12], 4)); print(np.round(ref["r_coarse"][:3, :12], 4))
