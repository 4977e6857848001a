import sys, glob, pickle, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
from oracle import spand_oracle as orc
import importlib.util
spec = importlib.util.spec_from_file_location("dm", "tools/dbg_multi.py")
src = open("tools/dbg_multi.py").read().split("bad = 0")[0]
ns = {}
exec(compile(src, "dbg_multi", "exec"), ns)
run = ns["run"]
bad = 0
for f in sorted(glob.glob("gpurun_out/wave_*.pkl")):
    d = pickle.load(open(f, "rb"))
    pan = [p for p in d["panels"]]
    keep = [i for i, p in enumerate(pan) if p.shape[0] > 0 and p.shape[1] > 0]
    pan = [pan[i] for i in keep]; gs = [d["groups"][i] for i in keep]
    if not pan: continue
    for rep in range(30):
        ev, blks = run(pan, gs, d["eps"], d["code"], np.nan)
        for i, a in enumerate(pan):
            ref = orc.sparsify_panel(a, d["eps"], ["first", "second-full", "second-superfine"][d["code"]])
            if ev[i, 4] != ref["rank_c"]:
                bad += 1; print(f, rep, i, a.shape, gs[i], ev[i, 4], ref["rank_c"], flush=True)
print("bad", bad)
