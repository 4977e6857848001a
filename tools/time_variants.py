"""Factorize time of the headline config under a few switches.

    python tools/time_variants.py [config] [levels]

Prints, per variant, the mean of 3 factorizations (after one warm-up) and
the engine's host timings (symbolic, plan, collect)."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2007_00789_b200 as sp
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    a, b, lv = sp.baseline_problem(name)
    if len(sys.argv) > 2:
        lv = int(sys.argv[2])
    h = sp.build_hierarchy(a, lv)
    for label, kw in (("digest_off", {"digest": False}), ("digest_on", {"digest": True}),
                      ("digest_off_2", {"digest": False})):
        sp.factorize(a, h, 0.01, "second-full", **kw)
        ts, tim = [], None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = sp.factorize(a, h, 0.01, "second-full", **kw)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            tim = f.timings
        print(json.dumps({"variant": label, "factorize_s": float(np.mean(ts)),
                          "timings": {k: round(v, 4) if isinstance(v, float) else v
                                      for k, v in tim.items()}}), flush=True)
        del f


if __name__ == "__main__":
    main()
