"""Shape statistics of the grouped-GEMM launches of the first factorization
level (host only: the first level's geometry does not depend on any rank).

    python tools/gemm_level_stats.py [C4] [15]

Per launch: tiles, targets, segments, useful FLOPs (2 r c K per segment) and
the FLOPs the tile kernel issues with the planner's tile shapes and with
64x64 tiles only (padding included)."""
import sys
import ctypes
sys.path.insert(0, '.')
import numpy as np
import paper_2007_00789_b200 as sp
from paper_2007_00789_b200 import engine as E

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 15
a, b, lv = sp.baseline_problem(name)
h = sp.build_hierarchy(a, levels)
sym = E.NativePlan(a, h, 0)
lib, vp = sym._lib, sym._vp
lib.spand_plan_emit_begin.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4
lib.spand_plan_emit_next.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.spand_plan_chunk.argtypes = [ctypes.c_void_p] * 3
POOL = 1 << 40
lib.spand_plan_emit_begin(sym.h, POOL, 2 << 40, 3 << 40, 4 << 40)
sizes = np.zeros(3, dtype=np.int64)
lib.spand_plan_emit_next(sym.h, vp(sizes))
plen, nlau, _ = (int(x) for x in sizes)
prog = np.zeros(max(plen, 1), dtype=np.int64)
lau = np.empty((nlau, 16), dtype=np.int64)
lib.spand_plan_chunk(sym.h, vp(prog), vp(lau))
m0 = np.concatenate([sym.m0, [sym.fcap]]).astype(np.int64)
bi, bj = np.asarray(sym.bi), np.asarray(sym.bj)


def dims(row):
    rc, cc, rs, cs, rn, cn = (int(x) for x in row[1:7])
    r = max(0, m0[rc] - rs)
    c = max(0, m0[cc] - cs)
    if rn >= 0:
        r = min(r, rn)
    if cn >= 0:
        c = min(c, cn)
    return r, c


tot_u = tot_x = tot_64 = 0
SHAPE = [(64, 64), (64, 16), (32, 32), (16, 16), (16, 64), (64, 32), (32, 64)]


def shape(mm, nn):   # planner.h tile_shape
    if mm <= 16 and nn <= 16:
        return 3
    if nn <= 16:
        return 1
    if mm <= 16:
        return 4
    if mm <= 32 and nn <= 32:
        return 2
    if nn <= 32:
        return 5
    if mm <= 32:
        return 6
    return 0


for li, rec in enumerate(lau):
    typ, cnt, ao, bo, co = (int(v) for v in rec[:5])
    if typ != 3:
        continue
    bT, lower, tri, compact = int(rec[5]), int(rec[6]), int(rec[7]), int(rec[10])
    tiles = prog[ao:ao + cnt]
    tgt = (tiles >> 32).astype(np.int64)
    nt = int(tgt.max()) + 1
    T = prog[bo:bo + 8 * (nt + 1)].reshape(-1, 8)
    useful = issued = issued64 = 0
    ks, rs, cs, nseg = [], [], [], []
    for t in np.unique(tgt).tolist():   # this launch's targets (one tile shape)
        r, c = dims(T[t])
        sb, se = int(T[t, 7]), int(T[t + 1, 7])
        nseg.append(se - sb)
        rs.append(r)
        cs.append(c)
        for s in range(sb, se):
            if compact:
                e = int(prog[co + s])
                K = int(m0[bj[e >> 32]])   # A block's columns
            else:
                ar = prog[co + 14 * s: co + 14 * s + 7]
                K = dims(ar)[1]
            ks.append(K)
            useful += 2 * r * c * K
            tm, tn = SHAPE[shape(r, c)]
            issued += -(-r // tm) * -(-c // tn) * 2 * tm * tn * ((K + 15) // 16 * 16)
            issued64 += -(-r // 64) * -(-c // 64) * 2 * 64 * 64 * ((K + 15) // 16 * 16)
    tot_u += useful
    tot_x += issued
    tot_64 += issued64
    q = lambda v: np.percentile(v, [50, 90, 99]).astype(int).tolist()  # noqa: E731
    print(f"launch {li}: shape {SHAPE[tri >> 4]} tiles {cnt} targets {len(rs)} segs {len(ks)} bT {bT} tri {tri} "
          f"rows p50/90/99 {q(rs)} cols {q(cs)} K {q(ks)} segs/target {q(nseg)} "
          f"useful {useful / 1e9:.1f} GF issued {issued / 1e9:.1f} GF ({useful / max(issued, 1):.0%}; "
          f"64x64 only: {issued64 / 1e9:.1f} GF)")
print(f"level 1: useful {tot_u / 1e9:.1f} GF, issued {tot_x / 1e9:.1f} GF "
      f"(64x64 tiles only: {tot_64 / 1e9:.1f} GF); K padded to 16, triangular bounds ignored")
