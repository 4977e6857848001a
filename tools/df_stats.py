import sys, re, collections
import numpy as np
lines = [l for l in open(sys.argv[1]) if l.startswith("[df]")]
S = collections.defaultdict(list)
for l in lines:
    for k, v in re.findall(r"(\w+) (\d+)", l[4:]):
        S[k].append(int(v))
for k in ("wait", "item", "chunk", "disp", "flush", "items", "chunks"):
    a = np.array(S[k]); print(k, "sum", a.sum(), "mean", round(a.mean(), 1), "max", a.max())
