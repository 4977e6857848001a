"""Device factorization engine: host level scheduler + batched sm_100a kernels.

Restates the reference driver (`/root/reference/pkg/src/spdkit/factorize.py`
`EliminationState` :51-239 and `factorize` :285-366) as three stages:

1. SYMBOLIC (host, once).  The block structure of the trailing matrix does
   not depend on the ranks the sparsification finds (ranks only shrink the
   live part of a cluster, `dofs[n_fine:]`, factorize.py:187-190), so the
   whole schedule is computed up front: per level the interior batch, the
   fill pattern and the grouped Schur targets (every same-level interior
   adjacent to a target block contributes one K-segment), the rescale batch
   and the sparsify WAVES (an interface waits for every adjacent interface
   with a smaller id, factorize.py:323; same-wave interfaces are
   independent).  Clusters that the reference drops (rank 0) simply have
   zero live size here; their later operators are filtered at collection.

2. NUMERIC (device, no host round trip).  Every dense matrix lives at its
   cluster pair's original size in one pool, column-major; the live window
   is read from the device ``off`` array that the RRQR kernel advances.  Per
   level: batched potrf -> trtri -> TRSM as DMMA GEMM with the explicit
   inverse -> one grouped DMMA GEMM for all Schur/fill updates; then (outside
   the skip window) batched rescale potrf/trtri + two GEMM passes
   (Z_i^-1 B Z_j^-T); then one cooperative RRQR launch per wave.  Finally
   the leftover clusters are assembled into one dense block and factored.

3. COLLECT (one sync).  Events (ranks, fine counts) and potrf infos come
   back; the host replays the offsets to build the operator list in the
   reference's order with device views of the payloads, the permutation,
   diagnostics and nnz_factor (counted on the device).
"""

import hashlib
import time

import numpy as np

from . import _lib
from .dense import SCHEME_CODE, SchemeKind
from .device import dev, ptr, require_cuda, stream, to_dev, to_dev_async
from .errors import NotSPD
from .kernels import Geometry, TILE, opnd
from .schemes import (Elimination, ErrorCorrection, MatView, Orthogonal,
                      Scaling)

import os as _os

WAVE_LOG = None      # set to [] to record per-wave CUDA events (profiling)
EVENT_ROW = 12
MAX_PANEL_ROWS = 6144


class NativePlan:
    """Handle on the C++ level scheduler (csrc/planner.cpp).

    ``meta`` decodes the scheduler's structure export into per-level
    records used by ``collect`` (operator assembly on the host)."""

    def __init__(self, a, h, skip_levels, cap_override=0):
        import ctypes
        t0 = time.perf_counter()
        lib = _lib.load()
        self.ncl = ncl = len(h.clusters)
        self.m0 = np.array([c.dofs.size for c in h.clusters], dtype=np.int64)
        self.depth = np.array([c.depth for c in h.clusters], dtype=np.int32)
        self.dofs = [np.asarray(c.dofs, dtype=np.int64) for c in h.clusters]
        self.cluster_of = h.cluster_of
        self.levels = h.levels
        rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.row_ptr))
        ci, cj = h.cluster_of[rows], h.cluster_of[a.col_idx]
        up = ci <= cj
        keys = np.ascontiguousarray(np.unique(ci[up] * ncl + cj[up]), dtype=np.int64)
        vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        lib.spand_plan_create.restype = ctypes.c_void_p
        lib.spand_plan_create.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_int]
        lib.spand_plan_destroy.argtypes = [ctypes.c_void_p]
        for nm, n in (("spand_plan_sizes", 2), ("spand_plan_program", 3),
                      ("spand_plan_meta", 2)):
            getattr(lib, nm).argtypes = [ctypes.c_void_p] * n
        lib.spand_plan_emit.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4
        self.h = ctypes.c_void_p(lib.spand_plan_create(
            ncl, vp(self.m0), vp(self.depth), int(h.levels), int(skip_levels),
            keys.size, vp(keys), int(cap_override)))
        self._lib = lib
        self._vp = vp
        self.sizes()
        self._decode_meta()
        self.seconds = time.perf_counter() - t0

    def __del__(self):
        try:
            self._lib.spand_plan_destroy(self.h)
        except Exception:
            pass

    def sizes(self):
        out = np.zeros(16, dtype=np.int64)
        self._lib.spand_plan_sizes(self.h, self._vp(out))
        (self.pool_size, self.fac_size, self.temp_size, self.n_events, self.n_info,
         self.n_ctr, self.nblocks, self.nlevels, self.fcap, self.f_off,
         self.flinv_off, self.nfinal, self.prog_len, self.n_launch,
         self.meta_len, _) = [int(x) for x in out]

    def emit(self, pool_base, fac_base, temp_base, ctr_base):
        self._lib.spand_plan_emit(self.h, pool_base, fac_base, temp_base, ctr_base)
        self.sizes()

    def program(self):
        prog = np.zeros(max(self.prog_len, 1), dtype=np.int64)
        lau = np.zeros(max(self.n_launch, 1) * 16, dtype=np.int64)
        self._lib.spand_plan_program(self.h, self._vp(prog), self._vp(lau))
        return prog, lau.reshape(-1, 16)[:self.n_launch]

    def _decode_meta(self):
        meta = np.zeros(max(self.meta_len, 1), dtype=np.int64)
        self._lib.spand_plan_meta(self.h, self._vp(meta))
        ncl, nb, nlev, nfin, nfinb = (int(x) for x in meta[:5])
        i = 9
        self.bi = meta[i:i + nb]; i += nb
        self.bj = meta[i:i + nb]; i += nb
        self.boff = meta[i:i + nb]; i += nb
        self.elim_linv = meta[i:i + ncl]; i += ncl
        self.bid = {(int(x), int(y)): k for k, (x, y) in enumerate(zip(self.bi, self.bj))}
        m = meta.tolist()
        recs = []
        for _ in range(nlev):
            level, skipped, nint, nact, nwaves = m[i:i + 5]; i += 5
            elim = []
            for _ in range(nint):
                s, nn = m[i], m[i + 1]; i += 2
                elim.append((s, tuple(m[i:i + nn]))); i += nn
            act = []
            for _ in range(nact):
                p, wv, lo, li, qo, sl, nn = m[i:i + 7]; i += 7
                act.append((p, wv, lo, li, qo, sl, tuple(m[i:i + nn]))); i += nn
            recs.append({"level": level, "skipped": bool(skipped), "elim": elim,
                         "active": act, "nwaves": nwaves})
        self.level_recs = recs
        self.final = m[i:i + nfin]; i += nfin
        self.final_blocks = m[i:i + nfinb]


class Engine:
    def __init__(self, a, h, eps, scheme, skip_levels):
        self.t = require_cuda()
        self.a, self.h = a, h
        self.eps, self.scheme, self.skip = eps, scheme, skip_levels
        self.sym = NativePlan(a, h, skip_levels,
                              int(_os.environ.get("SPAND_RRQR_CAP", "0")))
        self.timings = {"symbolic_s": self.sym.seconds}

    # -------------------------------------------------------------- numeric
    def run(self):
        """Allocate, emit the native program, upload it once, launch it."""
        t = self.t
        sym = self.sym
        m0 = sym.m0
        ncl = sym.ncl
        tstart = time.perf_counter()
        self.F = ncl
        self.fcap = sym.fcap
        self.geo = geo = Geometry(np.concatenate([m0, [sym.fcap]]).astype(np.int32))
        d = dev()
        self.pool = pool = t.zeros(max(sym.pool_size, 1), dtype=t.float64, device=d)
        self.facbuf = fac = t.zeros(max(sym.fac_size, 1), dtype=t.float64, device=d)
        self.boff = sym.boff
        self._scatter_a()
        self.events = t.zeros(max(sym.n_events, 1) * EVENT_ROW, dtype=t.int64, device=d)
        self.info = t.zeros(max(sym.n_info, 1), dtype=t.int32, device=d)
        ctr = t.zeros(max(sym.n_ctr, 1), dtype=t.int32, device=d)
        pb, fb = pool.data_ptr(), fac.data_ptr()
        sym.emit(pb, fb, 0, ctr.data_ptr())          # sizing pass (temp size)
        temp = t.empty(max(sym.temp_size, 1), dtype=t.float64, device=d)
        sym.emit(pb, fb, temp.data_ptr(), ctr.data_ptr())
        prog, launches = sym.program()
        self.timings["plan_s"] = time.perf_counter() - tstart
        progd = to_dev_async(prog)
        base = progd.data_ptr()
        st = stream()
        gm0, goff = ptr(geo.m0), ptr(geo.off)
        ib, evb = self.info.data_ptr(), self.events.data_ptr()
        import ctypes
        P = lambda off: ctypes.c_void_p(base + 8 * int(off))  # noqa: E731
        for rec in launches:
            typ, cnt, ao, bo, co, x0, x1, x2 = (int(v) for v in rec[:8])
            if typ == 1:
                _lib.call("spand_potrf_batched", cnt, P(ao), gm0, goff,
                          ctypes.c_void_p(ib + 4 * x0), st)
            elif typ == 2:
                _lib.call("spand_trtri_tiles", cnt, P(ao), gm0, goff, st)
            elif typ == 3:
                alpha = float(np.int64(rec[8]).view(np.float64))
                beta = float(np.int64(rec[9]).view(np.float64))
                _lib.call("spand_gemm_grouped", cnt, P(ao), P(bo), P(co), gm0, goff,
                          alpha, beta, x0, x1, st)
            elif typ == 4:
                _lib.call("spand_copy_batched", cnt, P(ao), gm0, goff, st)
            elif typ == 5:
                if WAVE_LOG is not None:
                    e0 = t.cuda.Event(enable_timing=True)
                    e1 = t.cuda.Event(enable_timing=True)
                    e0.record()
                _lib.call("spand_rrqr_wave", cnt, x0, x1, P(ao), P(bo), gm0, goff,
                          float(self.eps), SCHEME_CODE[self.scheme],
                          ctypes.c_void_p(evb), st)
                if WAVE_LOG is not None:
                    e1.record()
                    WAVE_LOG.append((cnt, x0, x1, e0, e1))
            elif typ == 6:
                _lib.call("spand_assemble_final", cnt, P(ao), x0, P(bo), gm0, goff,
                          x1, ctypes.c_void_p(fb + 8 * x2), st)
            else:
                raise RuntimeError(f"unknown launch type {typ}")
        self._keep_run = (temp, ctr, progd)
        t.cuda.synchronize()
        self.timings["device_s"] = time.perf_counter() - tstart

    def _scatter_a(self):
        """Initial blocks from the entries of A (factorize.py:61-96).

        The (pool offset, value) pairs are cached on the matrix's device
        cache per hierarchy, so refactorizing resident inputs does no
        host->device traffic."""
        sym, a = self.sym, self.a
        key = ("scatter", id(self.h), sym.pool_size)
        cached = a._dev.get(key) if a._dev is not None else None
        if cached is not None and cached[0] is self.h:
            self.pool[cached[1]] = cached[2]
            return
        n = a.n
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.row_ptr))
        cols = a.col_idx
        cl = sym.cluster_of
        slot = np.empty(n, dtype=np.int64)
        for c, dd in enumerate(sym.dofs):
            slot[dd] = np.arange(dd.size)
        ci, cj = cl[rows], cl[cols]
        up = ci <= cj
        ci, cj, r, c = ci[up], cj[up], rows[up], cols[up]
        keys = ci * sym.ncl + cj
        kk = sym.bi * sym.ncl + sym.bj
        order = np.argsort(kk)
        pos = order[np.searchsorted(kk[order], keys)]
        where = sym.boff[pos] + slot[r] + slot[c] * sym.m0[ci]
        vals = a.values[up]
        wd, vd = to_dev_async(where, np.int64), to_dev_async(vals, np.float64)
        self.pool[wd] = vd
        if a._dev is not None:
            a._dev[key] = (self.h, wd, vd)

    # --------------------------------------------------------------- collect
    def collect(self):
        t = self.t
        sym = self.sym
        m0 = sym.m0
        t0 = time.perf_counter()
        ev = self.events.cpu().numpy().reshape(-1, EVENT_ROW)
        if np.any(ev[:, 9] != 0):
            raise RuntimeError("RRQR group barrier watchdog fired (kernel bug)")
        # first non-SPD pivot in operator order (info slots follow launch order)
        iv = self.info.cpu().numpy()
        bad = np.flatnonzero(iv)
        if bad.size:
            raise NotSPD(int(iv[bad[0]]) - 1)
        off = np.zeros(sym.ncl, dtype=np.int64)
        pool, fac = self.pool, self.facbuf
        ops, perm_parts, diags = [], [], []
        views = []          # for the nonzero count: (MatView, op index)
        dofs = sym.dofs

        def live(c):
            return dofs[c][off[c]:]

        def bview(i, j, r0, c0, rows, cols, trans=False):
            b = int(sym.boff[sym.bid[(i, j)]])
            return MatView(pool, b + r0 + c0 * m0[i], m0[i], rows, cols, trans)

        def fview(at, c, size):
            return MatView(fac, at + off[c] + off[c] * m0[c], m0[c], size, size)

        scheme = self.scheme
        # structural apply phases (see apply.py): forward per level
        # [G-T][G-A]([D]([Q-T][E-A]) per wave); backward mirrored
        recs = sym.level_recs
        cnt = [2 + (0 if r["skipped"] else 1 + 2 * r["nwaves"]) for r in recs]
        fbase = np.concatenate([[0], np.cumsum(cnt)]).astype(int)
        bbase = [1 + int(sum(cnt[i + 1:])) for i in range(len(recs))]
        self.n_phases = int(fbase[-1]) + 1

        def phases(ri, kind, wave=0):
            r, fb, bb = recs[ri], int(fbase[ri]), bbase[ri]
            nw = 0 if r["skipped"] else r["nwaves"]
            if kind == "G":
                return ({"T": fb, "A": fb + 1},
                        {"A": bb + (2 * nw + 1 if not r["skipped"] else 0),
                         "T": bb + (2 * nw + 2 if not r["skipped"] else 1)})
            if kind == "D":
                return ({"T": fb + 2}, {"T": bb + 2 * nw})
            back = bb + 2 * (nw - 1 - wave)
            return ({"T": fb + 3 + 2 * wave, "A": fb + 4 + 2 * wave},
                    {"A": back, "T": back + 1})

        # apply records in the cluster-contiguous (permuted) numbering used by
        # the fast apply plan (fastplan.py): cluster c's slots live at
        # cstart[c] + [off[c], m0[c])
        cstart = np.concatenate([[0], np.cumsum(m0)[:-1]]).astype(np.int64)
        self.cstart = cstart
        arecs = []
        self.arecs = arecs

        def pst(c):
            return int(cstart[c] + off[c])

        for ri, rec in enumerate(sym.level_recs):
            lvl = rec["level"]
            nint, ndofs = 0, 0
            for s, nbrs in rec["elim"]:
                ns = m0[s] - off[s]
                if ns == 0:
                    continue
                nint += 1
                ndofs += ns
                wl = [w for w in nbrs if m0[w] - off[w] > 0]
                w_dofs = (np.concatenate([live(w) for w in wl]) if wl
                          else np.empty(0, np.int64))
                pv, r0 = [], 0
                for w in wl:
                    nw = m0[w] - off[w]
                    pv.append((bview(w, s, off[w], off[s], nw, ns), r0))
                    r0 += nw
                low = bview(s, s, off[s], off[s], ns, ns)
                linv = fview(int(sym.elim_linv[s]), s, ns)
                op = Elimination(live(s), w_dofs, low, pv, linv=linv)
                op._phases = phases(ri, "G")
                ops.append(op)
                arecs.append(("G", op._phases, pst(s), int(ns), linv,
                              [(pst(w), int(v.rows), v) for w, (v, _) in zip(wl, pv)]))
                perm_parts.append(live(s))
            faces = []
            if not rec["skipped"]:
                act = [x for x in rec["active"] if m0[x[0]] - off[x[0]] > 0]
                for p, wv, lo, li, qo, sl, nb in act:
                    mp = m0[p] - off[p]
                    op = Scaling(live(p), fview(lo, p, mp), linv=fview(li, p, mp))
                    op._phases = phases(ri, "D")
                    ops.append(op)
                    arecs.append(("D", op._phases, pst(p), int(mp), op.linv_view))
                for p, wv, lo, li, qo, sl, nb in act:
                    e = ev[sl]
                    mp, k_stop, k_c, rf2, n_fine = (int(e[1]), int(e[3]), int(e[4]),
                                                    int(e[5]), int(e[6]))
                    assert mp == m0[p] - off[p], "event / host offset mismatch"
                    old = live(p)
                    q = MatView(fac, qo, max(mp, 1), mp, mp, rot=k_c if mp else 0)
                    qop = Orthogonal(old, q)
                    qop._phases = phases(ri, "Q", wv)
                    ops.append(qop)
                    arecs.append(("Q", qop._phases, pst(p), int(mp), q))
                    if scheme is SchemeKind.SECOND_ORDER_FULL:
                        ncorr = n_fine
                    elif scheme is SchemeKind.SECOND_ORDER_SUPERFINE:
                        ncorr = k_stop - k_c
                    else:
                        ncorr = 0
                    wl = [w for w in nb if m0[w] - off[w] > 0]
                    ntot = int(sum(m0[w] - off[w] for w in wl))
                    if ncorr and ntot:
                        evs, c0 = [], 0
                        for w in wl:
                            nw = m0[w] - off[w]
                            if w > p:
                                v = bview(p, w, off[p], off[w], ncorr, nw)
                            else:
                                v = bview(w, p, off[w], off[p], nw, ncorr, trans=True)
                            evs.append((v, c0))
                            c0 += nw
                        w_dofs = np.concatenate([live(w) for w in wl])
                        eop = ErrorCorrection(old[:ncorr], w_dofs, evs)
                        eop._phases = qop._phases
                        ops.append(eop)
                        arecs.append(("E", qop._phases, pst(p), int(ncorr),
                                      [(pst(w), int(m0[w] - off[w]), v)
                                       for w, (v, _) in zip(wl, evs)]))
                    if n_fine:
                        perm_parts.append(old[:n_fine])
                    faces.append({"cluster": int(p), "size_before": int(mp),
                                  "size_after": int(k_c), "rank_f2": int(rf2),
                                  "eta_stop": float(np.int64(e[7]).view(np.float64)),
                                  "r11": float(np.int64(e[8]).view(np.float64)),
                                  "k_stop": int(k_stop), "n_cols": int(e[2])})
                    off[p] += n_fine
            digest = hashlib.sha256(repr([(f["cluster"], f["size_before"],
                                           f["size_after"], f["rank_f2"])
                                          for f in faces]).encode()).hexdigest()
            diags.append({"level": int(lvl), "interior_clusters": nint,
                          "interior_dofs": int(ndofs), "skipped": bool(rec["skipped"]),
                          "interfaces": [{k: f[k] for k in ("cluster", "size_before",
                                                            "size_after", "rank_f2")}
                                         for f in faces],
                          "margins": faces,
                          "digest": digest})
        fin = [c for c in sym.final if m0[c] - off[c] > 0]
        total = int(sum(m0[c] - off[c] for c in fin))
        if total:
            foff = sym.fcap - total
            low = MatView(fac, sym.f_off + foff + foff * sym.fcap, sym.fcap, total, total)
            linv = MatView(fac, sym.flinv_off + foff + foff * sym.fcap, sym.fcap,
                           total, total)
            fd = np.concatenate([live(c) for c in fin])
            fop = Elimination(fd, np.empty(0, np.int64), low, [], linv=linv)
            fop._phases = ({"T": self.n_phases - 1, "A": self.n_phases - 1},
                           {"T": 0, "A": 0})
            ops.append(fop)
            fidx = np.concatenate([np.arange(pst(c), cstart[c] + m0[c]) for c in fin])
            arecs.append(("F", fop._phases, fidx, total, linv))
            perm_parts.append(fd)
        perm = (np.concatenate(perm_parts) if perm_parts else np.empty(0, np.int64))
        nnz = self._count(ops)
        self.timings["collect_s"] = time.perf_counter() - t0
        return ops, perm, {"levels": diags, "final_block": total}, nnz

    def _count(self, ops):
        t = self.t
        rows = []
        for op in ops:
            vs = []
            if isinstance(op, Elimination):
                vs = [op._lower] + [v for v, _ in op.panel_views]
            elif isinstance(op, Scaling):
                vs = [op._lower]
            elif isinstance(op, Orthogonal):
                vs = [op.q_view]
            else:
                vs = [v for v, _ in op.e_views]
            for v in vs:
                if v.rows and v.cols:
                    rows.append([v.addr, v.ld, v.rows, v.cols])
        if not rows:
            return 0
        vd = to_dev(np.asarray(rows, dtype=np.int64))
        out = t.zeros(len(rows), dtype=t.int64, device=dev())
        _lib.call("spand_count_nonzero", len(rows), ptr(vd), ptr(out), stream())
        return int(out.sum().item())


def ctypes_ptr(addr):
    import ctypes
    return ctypes.c_void_p(int(addr))


def run_factorization(a, h, eps, scheme, skip_levels, collect_local_errors=False):
    from .factorize import Factorization
    t0 = time.perf_counter()
    eng = Engine(a, h, eps, scheme, skip_levels)
    eng.run()
    ops, perm, diag, nnz = eng.collect()
    eng.timings["total_s"] = time.perf_counter() - t0
    f = Factorization(ops=ops, perm=perm, n=a.n, eps=float(eps), scheme=scheme,
                      skip_levels=int(skip_levels), nnz_factor=int(nnz),
                      diagnostics=diag,
                      _keep=(eng.pool, eng.facbuf, eng.geo), timings=eng.timings)
    perm_c = np.concatenate(eng.sym.dofs) if eng.sym.dofs else np.empty(0, np.int64)
    arecs, nph = eng.arecs, eng.n_phases

    def factory():
        from .fastplan import FastPlan
        return FastPlan(a.n, perm_c, arecs, nph)

    f._plan_factory = factory
    return f
