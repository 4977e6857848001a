"""Host cost of the native collector (csrc/collect.cpp) on C4-L15.

    python tools/collect_bench.py dump    # GPU box: factorize once, save the events
    python tools/collect_bench.py time    # anywhere: time spand_collect_create /
                                          # spand_collect_apply on the saved events

The collector only needs the plan (host) and the per-interface events
(ranks), so its cost can be measured and tuned without a GPU."""
import ctypes
import hashlib
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine as E

EV = "gpurun_out/events_c4_l15.npy"
a, b, lv = sp.baseline_problem("C4")
h = sp.build_hierarchy(a, 15)
if sys.argv[1] == "dump":
    keep = {}
    orig = E.Engine.collect

    def col(self):
        keep["ev"] = self.events.cpu().numpy().copy()
        return orig(self)
    E.Engine.collect = col
    sp.factorize(a, h, 1e-2, "second-full")
    np.save(EV, keep["ev"])
    print("saved", keep["ev"].shape)
    sys.exit(0)

ev = np.ascontiguousarray(np.load(EV))
sym = E.NativePlan(a, h, 4)
lib, vp = sym._lib, sym._vp
# the collector reads the per-level records the emission fills in
lib.spand_plan_emit_begin.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4
lib.spand_plan_emit_next.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.spand_plan_emit_begin(sym.h, 1 << 40, 2 << 40, 3 << 40, 4 << 40)
sizes = np.zeros(3, dtype=np.int64)
while lib.spand_plan_emit_next(sym.h, vp(sizes)):
    pass
lib.spand_collect_create.restype = ctypes.c_void_p
lib.spand_collect_create.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
lib.spand_collect_destroy.argtypes = [ctypes.c_void_p]
lib.spand_collect_apply.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4 + [ctypes.c_void_p]
lib.spand_collect_apply_get.argtypes = [ctypes.c_void_p] * 3
for rep in range(4):
    t0 = time.perf_counter()
    ch = lib.spand_collect_create(sym.h, vp(ev), E.SCHEME_CODE[sp.SchemeKind.from_string("second-full")])
    t1 = time.perf_counter()
    out = np.zeros(4, dtype=np.int64)
    rc = lib.spand_collect_apply(ch, 1 << 40, 2 << 40, 3 << 40, 4 << 40, None, vp(out))
    t2 = time.perf_counter()
    img = np.empty(int(out[0]), dtype=np.int64)
    ph = np.zeros((int(out[1] + out[2]), 10), dtype=np.int64)
    lib.spand_collect_apply_get(ch, vp(img), vp(ph))
    t3 = time.perf_counter()
    lib.spand_collect_destroy(ch)
    dig = hashlib.sha256(img.tobytes() + ph.tobytes()).hexdigest()[:16]
    print(f"create {1e3 * (t1 - t0):.1f} ms  apply {1e3 * (t2 - t1):.1f} ms  get {1e3 * (t3 - t2):.1f} ms"
          f"  image {img.nbytes / 1e6:.1f} MB  rc {rc}  digest {dig}")
ch = lib.spand_collect_create(sym.h, vp(ev), 2)
sz = np.zeros(8, dtype=np.int64)
lib.spand_collect_sizes.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.spand_collect_sizes(ch, vp(sz))
print("nops nsegs nperm ndiag nlsum nviews final nfine:", sz.tolist())
