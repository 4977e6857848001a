import sys, glob, pickle, numpy as np
sys.path.insert(0, '.')
sys.argv = [sys.argv[0]]
import tools.dbg_multi as dm  # noqa (runs its own trials with count default 20)
