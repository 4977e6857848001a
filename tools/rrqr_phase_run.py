"""Run one C4 factorization with the phase-instrumented RRQR build
(tools/build_variant.sh phases -DSPAND_RRQR_PHASES); the kernel prints
per-phase kilocycles for panels of >= 1000 rows."""
import os, sys
sys.path.insert(0, '.')
os.environ["SPAND_LIB_PATH"] = os.path.abspath("paper_2007_00789_b200/variants/libspand_phases.so")
import paper_2007_00789_b200 as sp
levels = int(sys.argv[1]) if len(sys.argv) > 1 else 15
a, b, lv = sp.baseline_problem("C4")
h = sp.build_hierarchy(a, levels)
f = sp.factorize(a, h, 1e-2, "second-full")
print("factorize", f.timings)
