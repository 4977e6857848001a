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
from .device import ARENA, dev, ptr, require_cuda, stream, to_dev, to_dev_async
from .errors import NotSPD
from .kernels import Geometry, TILE, opnd
from .schemes import (Elimination, ErrorCorrection, MatView, Orthogonal,
                      Scaling)

import os as _os
from collections.abc import Sequence

# launch record type -> entry point (csrc/launcher.cu spand_run_launches)
LAUNCH_NAMES = {1: "spand_potrf_batched", 2: "spand_trtri_tiles", 3: "spand_gemm_grouped",
                4: "spand_copy_batched", 5: "spand_rrqr_wave", 6: "spand_assemble_final",
                7: "spand_nk_rescale", 8: "spand_nk_basis", 9: "spand_nk_deflate",
                10: "spand_nk_qform", 11: "spand_digest_pieces", 12: "spand_gemm_kmask"}
WAVE_LOG = None      # set to [] to record per-wave CUDA events (profiling)
PROG_ARENA = None    # pinned staging of the program chunks (emission thread)
NK_RTOL = 1e-8       # rank threshold of the near-kernel basis (oracle NK_RTOL)
EVENT_ROW = 12
MAX_PANEL_ROWS = 24576   # rrqr.cu kMaxM (reflector in shared memory)


class NativePlan:
    """Handle on the C++ level scheduler (csrc/planner.cpp).

    ``meta`` decodes the scheduler's structure export into per-level
    records used by ``collect`` (operator assembly on the host)."""

    def __init__(self, a, h, skip_levels, cap_override=0, nk=0, digest=False):
        import ctypes
        t0 = time.perf_counter()
        lib = _lib.load()
        self.ncl = ncl = len(h.clusters)
        self.m0 = np.array([c.dofs.size for c in h.clusters], dtype=np.int64)
        self.depth = np.array([c.depth for c in h.clusters], dtype=np.int32)
        self.dofs = [np.asarray(c.dofs, dtype=np.int64) for c in h.clusters]
        self.cluster_of = h.cluster_of
        self.levels = h.levels
        vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        dcat = np.ascontiguousarray(np.concatenate(self.dofs) if self.dofs
                                    else np.zeros(1, np.int64), dtype=np.int64)
        dptr = np.zeros(ncl + 1, dtype=np.int64)
        np.cumsum(self.m0, out=dptr[1:])
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        cx = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        cof = np.ascontiguousarray(h.cluster_of, dtype=np.int64)
        keys = np.empty(max(cx.size, 1), dtype=np.int64)
        lib.spand_plan_pairs.restype = ctypes.c_int64
        lib.spand_plan_pairs.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 6
        npairs = lib.spand_plan_pairs(ncl, vp(rp), vp(cx), vp(cof), vp(dcat), vp(dptr), vp(keys))
        keys = keys[:npairs]
        lib.spand_plan_create.restype = ctypes.c_void_p
        lib.spand_plan_create.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_int]
        lib.spand_plan_destroy.argtypes = [ctypes.c_void_p]
        for nm, n in (("spand_plan_sizes", 2), ("spand_plan_program", 3),
                      ("spand_plan_meta", 2)):
            getattr(lib, nm).argtypes = [ctypes.c_void_p] * n
        lib.spand_plan_emit.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4 + [ctypes.c_int]
        self.h = ctypes.c_void_p(lib.spand_plan_create(
            ncl, vp(self.m0), vp(self.depth), int(h.levels), int(skip_levels),
            keys.size, vp(keys), int(cap_override)))
        self._lib = lib
        self._vp = vp
        lib.spand_plan_set_dofs.argtypes = [ctypes.c_void_p] * 3
        lib.spand_plan_set_dofs(self.h, vp(dcat), vp(dptr))
        gw = int(_os.environ.get("SPAND_GROUP_WEIGHT", "-1"))
        if gw >= 0:
            lib.spand_plan_set_group_weight.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                                        ctypes.c_double, ctypes.c_double]
            lib.spand_plan_set_group_weight(
                self.h, gw, float(_os.environ.get("SPAND_GROUP_EM", "1.25")),
                float(_os.environ.get("SPAND_GROUP_EN", "0.5")))
        cl = _os.environ.get("SPAND_RRQR_CLUSTER")
        if cl is not None:
            lib.spand_plan_set_cluster.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
            if lib.spand_plan_set_cluster(
                    self.h, int(cl), int(_os.environ.get("SPAND_RRQR_CLUSTER_MIN", "256"))) != 0:
                raise ValueError(f"SPAND_RRQR_CLUSTER={cl}: cluster size must be 0, 2, 4 or 8")
        if nk:
            if lib.spand_plan_set_nk(self.h, int(nk)) != 0:
                raise ValueError(f"at most 16 near-kernel vectors, got {nk}")
        self.digest_first = None
        if digest:
            lib.spand_plan_set_digest.restype = ctypes.c_int64
            lib.spand_plan_set_digest.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                                  ctypes.c_int64, ctypes.c_void_p]
            first = np.zeros(int(h.levels) + 1, dtype=np.int64)
            lib.spand_plan_set_digest(self.h, 1, 0, vp(first))
            self.digest_first = first
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
         self.meta_len, self.temp_bound) = [int(x) for x in out]

    def emit(self, pool_base, fac_base, temp_base, ctr_base, dry=False):
        self._lib.spand_plan_emit(self.h, pool_base, fac_base, temp_base, ctr_base,
                                  int(dry))
        self.sizes()

    def program(self):
        prog = np.zeros(max(self.prog_len, 1), dtype=np.int64)
        lau = np.zeros(max(self.n_launch, 1) * 16, dtype=np.int64)
        self._lib.spand_plan_program(self.h, self._vp(prog), self._vp(lau))
        return prog, lau.reshape(-1, 16)[:self.n_launch]

    def _decode_meta(self):
        """Block arrays (needed by every factorization); the per-level
        records are decoded lazily (tools and structural tests only)."""
        meta = np.zeros(max(self.meta_len, 1), dtype=np.int64)
        self._lib.spand_plan_meta(self.h, self._vp(meta))
        ncl, nb = (int(x) for x in meta[:2])
        i = 9
        self.bi = meta[i:i + nb]; i += nb
        self.bj = meta[i:i + nb]; i += nb
        self.boff = meta[i:i + nb]; i += nb
        self.elim_linv = meta[i:i + ncl]; i += ncl
        self._meta, self._meta_at, self._recs = meta, i, None

    @property
    def bid(self):
        return {(int(x), int(y)): k for k, (x, y) in enumerate(zip(self.bi, self.bj))}

    @property
    def level_recs(self):
        if self._recs is None:
            self._decode_levels()
        return self._recs

    @property
    def final(self):
        if self._recs is None:
            self._decode_levels()
        return self._final

    @property
    def final_blocks(self):
        if self._recs is None:
            self._decode_levels()
        return self._final_blocks

    def _decode_levels(self):
        meta, i = self._meta, self._meta_at
        nlev, nfin, nfinb = (int(x) for x in meta[2:5])
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
        self._recs = recs
        self._final = m[i:i + nfin]; i += nfin
        self._final_blocks = m[i:i + nfinb]


class Engine:
    def __init__(self, a, h, eps, scheme, skip_levels, near_kernel=None,
                 collect_local_errors=False, digest=False):
        self.t = require_cuda()
        self.a, self.h = a, h
        self.local_errors = bool(collect_local_errors)
        self.eps, self.scheme, self.skip = eps, scheme, skip_levels
        self.nk = near_kernel      # n x k host array (extension) or None
        self.sym = NativePlan(a, h, skip_levels,
                              int(_os.environ.get("SPAND_RRQR_CAP", "0")),
                              0 if near_kernel is None else near_kernel.shape[1],
                              digest=digest)
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
        self.events = t.zeros(max(sym.n_events, 1) * EVENT_ROW, dtype=t.int64, device=d)
        self.info = t.zeros(max(sym.n_info, 1), dtype=t.int32, device=d)
        ctr = t.zeros(2 * max(sym.n_ctr, 1), dtype=t.int32, device=d)   # {arrivals, release} per panel
        pb, fb = pool.data_ptr(), fac.data_ptr()
        temp = t.empty(max(sym.temp_bound, 1), dtype=t.float64, device=d)
        st = stream()
        gm0, goff = ptr(geo.m0), ptr(geo.off)
        ib, evb = self.info.data_ptr(), self.events.data_ptr()
        import ctypes
        lib = sym._lib
        vp = sym._vp
        # incremental emission: level l + 1 is planned on the host while the
        # device runs level l (all launches are asynchronous)
        lib.spand_plan_emit_begin.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4
        lib.spand_plan_emit_next.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.spand_plan_chunk.argtypes = [ctypes.c_void_p] * 3
        if sym.digest_first is not None:
            # trailing-matrix digest records {i, j, rows, cols, hash} per
            # (level, alive block), written by the type-11 launches
            nrec = int(sym.digest_first[-1])
            self.digest_rec = t.zeros(max(nrec, 1) * 5, dtype=t.int64, device=d)
            lib.spand_plan_set_digest(sym.h, 1, self.digest_rec.data_ptr(), None)
        lib.spand_plan_emit_begin(sym.h, pb, fb, temp.data_ptr(), ctr.data_ptr())
        # the next level is emitted on a helper thread (ctypes releases the
        # GIL) while this one uploads and launches the current level
        from concurrent.futures import ThreadPoolExecutor
        acc = {"plan": 0.0}

        def produce():
            # the chunk is written straight into pinned memory (PROG_ARENA:
            # used by this helper thread only, recycled after the run's sync)
            tp = time.perf_counter()
            sizes = np.zeros(3, dtype=np.int64)
            more = lib.spand_plan_emit_next(sym.h, vp(sizes))
            plen, nlau, used_ = (int(x) for x in sizes)
            prog_ = launches_ = None
            if nlau:
                stage = PROG_ARENA.take(8 * max(plen, 1)).view(t.int64)
                prog_ = stage.numpy()
                launches_ = np.empty((nlau, 16), dtype=np.int64)
                lib.spand_plan_chunk(sym.h, vp(prog_), vp(launches_))
                prog_ = (prog_, stage)
            acc["plan"] += time.perf_counter() - tp
            return more, prog_, launches_, used_

        global PROG_ARENA
        if PROG_ARENA is None:
            from .device import PinnedArena
            PROG_ARENA = PinnedArena()
        ex = ThreadPoolExecutor(1)
        # the first level is emitted while A's entries are scattered into the pool
        fut = ex.submit(produce)
        self._scatter_a()
        if self.nk is not None:
            # near-kernel coordinates in the cluster-contiguous numbering,
            # column-major n x k (vector v at nkbuf[v])
            perm_c = np.concatenate(sym.dofs)
            self.nkbuf = to_dev(np.ascontiguousarray(self.nk[perm_c].T))
        # block table of the compact Schur segments: {ptr, rc, cc} per block
        btab = np.stack([pb + 8 * np.asarray(sym.boff, dtype=np.int64),
                         np.asarray(sym.bi, dtype=np.int64),
                         np.asarray(sym.bj, dtype=np.int64)], axis=1)
        self._btab = to_dev_async(np.ascontiguousarray(btab))
        self._btab_p = ptr(self._btab)

        keep = []
        t_launch = 0.0
        with ex:
            while True:
                more, prog, launches, used = fut.result()
                if more:
                    fut = ex.submit(produce)
                if launches is not None:
                    tl = time.perf_counter()
                    prog, stage = prog
                    progd = t.empty(stage.shape, dtype=t.int64, device=d)
                    progd.copy_(stage, non_blocking=True)
                    keep.append(progd)
                    self._launch(launches, progd.data_ptr(), gm0, goff, ib, evb, fb, st, prog)
                    t_launch += time.perf_counter() - tl
                if not more:
                    break
        t_plan = acc["plan"]
        self.timings["launch_s"] = t_launch
        assert used <= sym.temp_bound, (used, sym.temp_bound)
        self.timings["plan_s"] = t_plan
        self._keep_run = (temp, ctr, keep)
        t.cuda.synchronize()
        ARENA.reset()   # every staged upload has completed
        PROG_ARENA.reset()
        self.timings["device_s"] = time.perf_counter() - tstart

    def _launch(self, launches, base, gm0, goff, ib, evb, fb, st, prog=None):
        if WAVE_LOG is None and _os.environ.get("SPAND_NATIVE_LAUNCH", "1") != "0":
            self._launch_native(launches, base, gm0, goff, ib, evb, fb, st)
            return
        import ctypes
        t = self.t
        P = lambda off: ctypes.c_void_p(base + 8 * int(off))  # noqa: E731
        for rec in launches:
            typ, cnt, ao, bo, co, x0, x1, x2 = (int(v) for v in rec[:8])
            if typ == 1:
                _lib.call("spand_potrf_batched", cnt, P(ao), gm0, goff,
                          ctypes.c_void_p(ib), x0, x1, st)
            elif typ == 2:
                _lib.call("spand_trtri_tiles", cnt, P(ao), gm0, goff, st)
            elif typ == 3:
                alpha = float(np.int64(rec[8]).view(np.float64))
                beta = float(np.int64(rec[9]).view(np.float64))
                if int(rec[11]):
                    # K-chunk masks (written by a type-12 record just before)
                    _lib.call("spand_gemm_grouped_masked", cnt, P(ao), P(bo), P(co), gm0, goff,
                              alpha, beta, x0, x1, x2, self._btab_p, int(rec[10]),
                              ctypes.c_void_p(int(rec[11])), P(bo + int(rec[12])), st)
                else:
                    _lib.call("spand_gemm_grouped", cnt, P(ao), P(bo), P(co), gm0, goff,
                              alpha, beta, x0, x1, x2, self._btab_p, int(rec[10]), st)
            elif typ == 12:
                _lib.call("spand_gemm_kmask", cnt, P(ao), P(bo), gm0, goff,
                          ctypes.c_void_p(x0), P(co), x1, st)
            elif typ == 4:
                _lib.call("spand_copy_batched", cnt, P(ao), gm0, goff, st)
            elif typ == 5:
                if WAVE_LOG is not None:
                    e0 = t.cuda.Event(enable_timing=True)
                    e1 = t.cuda.Event(enable_timing=True)
                    e0.record()
                flags = SCHEME_CODE[self.scheme] | (4 if self.local_errors else 0)
                if x2 > 1:
                    _lib.call("spand_rrqr_wave_clustered", cnt, x0, x1, x2, P(ao), P(bo),
                              gm0, goff, float(self.eps), flags, ctypes.c_void_p(evb), st)
                else:
                    _lib.call("spand_rrqr_wave", cnt, x0, x1, P(ao), P(bo), gm0, goff,
                              float(self.eps), flags, ctypes.c_void_p(evb), st)
                if WAVE_LOG is not None:
                    e1.record()
                    slots = [int(prog[ao + 16 * q + 10]) for q in range(cnt)] if prog is not None else []
                    WAVE_LOG.append((cnt, x0, x1, e0, e1, slots))
            elif typ in (7, 8, 9, 10):
                U, k = self.nkbuf, self.nkbuf.shape[0]
                if typ == 7:
                    _lib.call("spand_nk_rescale", cnt, P(ao), gm0, goff, ptr(U),
                              U.shape[1], k, x0, st)
                elif typ == 8:
                    _lib.call("spand_nk_basis", cnt, P(ao), P(bo), gm0, goff, ptr(U),
                              U.shape[1], k, NK_RTOL, st)
                elif typ == 9:
                    _lib.call("spand_nk_deflate", cnt, x0, P(ao), P(bo), gm0, goff, x1, st)
                else:
                    _lib.call("spand_nk_qform", cnt, x0, P(ao), ctypes.c_void_p(evb), x1, st)
            elif typ == 11:
                _lib.call("spand_digest_pieces", cnt, P(ao), gm0, goff, st)
            elif typ == 6:
                _lib.call("spand_assemble_final", cnt, P(ao), x0, P(bo), gm0, goff,
                          x1, ctypes.c_void_p(fb + 8 * x2), st)
            else:
                raise RuntimeError(f"unknown launch type {typ}")

    def _launch_native(self, launches, base, gm0, goff, ib, evb, fb, st):
        """All records of a program chunk issued by one native call
        (csrc/launcher.cu): no per-launch ctypes overhead on the host."""
        import ctypes
        recs = np.ascontiguousarray(launches, dtype=np.int64)
        if recs.size == 0:
            return
        counts = np.zeros(16, dtype=np.int64)
        U, ldu, nkv = None, 0, 0
        if self.nk is not None and hasattr(self, "nkbuf"):
            U, ldu, nkv = ptr(self.nkbuf), int(self.nkbuf.shape[1]), int(self.nkbuf.shape[0])
        mask = _lib.profile_mask(LAUNCH_NAMES)
        _lib.call("spand_run_launches", int(recs.shape[0]), recs.ctypes.data, int(base), gm0, goff,
                  ctypes.c_void_p(ib), ctypes.c_void_p(evb), int(fb), self._btab_p,
                  float(self.eps), SCHEME_CODE[self.scheme] | (4 if self.local_errors else 0),
                  U, ldu, nkv, float(NK_RTOL), mask, counts.ctypes.data, st)
        for typ, nm in LAUNCH_NAMES.items():
            if counts[typ]:
                _lib.COUNTS[nm] = _lib.COUNTS.get(nm, 0) + int(counts[typ])

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
        import ctypes
        lib = sym._lib
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        cx = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        cof = np.ascontiguousarray(sym.cluster_of, dtype=np.int64)
        where = np.empty(max(cx.size, 1), dtype=np.int64)
        lib.spand_plan_scatter.argtypes = [ctypes.c_void_p] * 5
        if lib.spand_plan_scatter(sym.h, sym._vp(rp), sym._vp(cx), sym._vp(cof),
                                  sym._vp(where)) != 0:
            raise RuntimeError("block of a nonzero of A missing from the symbolic structure")
        where = where[:cx.size]
        up = where >= 0
        where = where[up]
        vals = a.values[up]
        wd, vd = to_dev_async(where, np.int64), to_dev_async(vals, np.float64)
        self.pool[wd] = vd
        if a._dev is not None:
            a._dev[key] = (self.h, wd, vd)

    # --------------------------------------------------------------- collect
    def collect(self):
        """Operators, permutation, diagnostics and nnz from the native
        collector (csrc/collect.cpp), payloads as lazy device views."""
        import ctypes
        t0 = time.perf_counter()
        sym = self.sym
        lib = _lib.load()
        ev = self.events.cpu().numpy().reshape(-1, EVENT_ROW)
        if np.any(ev[:, 9] != 0):
            raise RuntimeError("RRQR group barrier watchdog fired (kernel bug)")
        # first non-SPD pivot in operator order (info slots follow launch order)
        iv = self.info.cpu().numpy()
        bad = np.flatnonzero(iv)
        if bad.size:
            raise NotSPD(int(iv[bad[0]]) - 1)
        vp = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        lib.spand_collect_create.restype = ctypes.c_void_p
        lib.spand_collect_create.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.spand_collect_destroy.argtypes = [ctypes.c_void_p]
        evc = np.ascontiguousarray(ev)
        ch = ctypes.c_void_p(lib.spand_collect_create(sym.h, vp(evc),
                                                      SCHEME_CODE[self.scheme]))
        self.collected = Collected(lib, ch, vp)
        col = self.collected
        t1 = time.perf_counter()
        stats = np.zeros(1, dtype=np.int64)
        lib.spand_collect_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.spand_collect_stats(ch, vp(stats))
        self.timings["rrqr_critical_steps"] = int(stats[0])
        # the apply image compiles on a host thread while the diagnostics and
        # the nonzero count below run (the first apply waits for it)
        from .fastplan import NativeApplyPlan
        perm_c = np.concatenate(sym.dofs) if sym.dofs else np.empty(0, np.int64)
        self.apply_plan = NativeApplyPlan(self.a.n, perm_c, col, self.pool, self.facbuf)
        ops = LazyOps(col, sym.dofs, self.pool, self.facbuf)
        t2 = time.perf_counter()
        # diagnostics (factorize.py:331-356) + margins of every decision
        diags = []
        by_level = {}
        dv = col.diag.copy()
        etas = dv[:, 5].view(np.float64).tolist()
        r11s = dv[:, 6].view(np.float64).tolist()
        entries = []
        for q, d in enumerate(col.diag.tolist()):
            li, p, mp, kc, rf2, eb, rb, ks, nc, _ = d
            entries.append({
                "cluster": p, "size_before": mp, "size_after": kc, "rank_f2": rf2,
                "eta_stop": etas[q], "r11": r11s[q], "k_stop": ks,
                "n_cols": nc})
            by_level.setdefault(li, []).append(entries[-1])
        if self.local_errors:
            errs = self._local_errors(col)
            for q, ent in enumerate(entries):
                ent["local_error"] = errs[q]
        digests = self._digests()
        for li, (lvl, nint, ndofs, skipped) in enumerate(col.lsum.tolist()):
            faces = by_level.get(li, [])
            digest = digests[li] if digests is not None else None
            diags.append({"level": lvl, "interior_clusters": nint,
                          "interior_dofs": ndofs, "skipped": bool(skipped),
                          "interfaces": [{k: f[k] for k in ("cluster", "size_before",
                                                            "size_after", "rank_f2",
                                                            "local_error") if k in f}
                                         for f in faces],
                          "margins": faces, "digest": digest})
        t3 = time.perf_counter()
        nnz = self._count(col.views)
        t4 = time.perf_counter()
        self.timings.update(collect_s=t4 - t0, collect_native_s=t1 - t0,
                            collect_apply_start_s=t2 - t1, collect_diag_s=t3 - t2,
                            collect_count_s=t4 - t3)
        return ops, col.perm, {"levels": diags, "final_block": col.final_total}, nnz

    def _digests(self):
        """Per-level trailing-matrix fingerprints (reference
        EliminationState.digest, factorize.py:222-229): sha256 over the
        level's alive blocks in key order of (i, j, rows, cols, h), h the
        device hash of the block's live window (dense_small.cu
        digest_kernel).  Identical trailing matrices -- e.g. across the
        three schemes, which differ only in their correction operators --
        give identical digests; the bytes differ from the reference's
        sha256 of the raw blocks (a different fingerprint of the same
        state)."""
        first = self.sym.digest_first
        if first is None:
            return None
        rec = self.digest_rec.cpu().numpy().reshape(-1, 5)
        out = []
        for k in range(len(first) - 1):
            r = rec[first[k]:first[k + 1]]
            r = r[(r[:, 2] > 0) & (r[:, 3] > 0)]
            out.append(hashlib.sha256(np.ascontiguousarray(r, dtype="<i8").tobytes())
                       .hexdigest())
        return out

    def _local_errors(self, col):
        """Spectral norm of the dropped term of every sparsification
        (reference `local_error`, schemes.py:321-340, from the norms of
        schemes.py:297-306): first order ||Q_f^T W||, full second order
        ||E||^2, superfine max(||E||^2, ||Q_f1^T W||).  The fine rows Q_f^T W
        are kept in the dead slots by the RRQR (flag 4); the norm is
        sqrt(lambda_max(F F^T)) on the device (diagnostics only)."""
        import ctypes
        t = self.t
        nd = col.diag.shape[0]
        out = [0.0] * nd
        if col.nfine == 0:
            return out
        fine = np.zeros((col.nfine, 8), dtype=np.int64)
        col.lib.spand_collect_fine.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        col.lib.spand_collect_fine(col.h, col.vp(fine))
        pool = self.pool
        code = SCHEME_CODE[self.scheme]
        starts = np.flatnonzero(np.r_[True, fine[1:, 0] != fine[:-1, 0]])
        ends = np.r_[starts[1:], fine.shape[0]]
        for s0, s1 in zip(starts, ends):
            q = int(fine[s0, 0])
            parts = []
            for _, _, off, ld, r, c, tr, _ in fine[s0:s1].tolist():
                # F is n_fine x (neighbour columns); a transposed block (w, p)
                # holds F's columns as rows of w
                parts.append(pool.as_strided((c, r), (ld, 1), off) if tr
                             else pool.as_strided((r, c), (1, ld), off))
            f = t.cat(parts, dim=1)
            rf2 = int(col.diag[q, 4])

            def spec(m):
                if m.shape[0] == 0 or m.shape[1] == 0:
                    return 0.0
                g = m @ m.t() if m.shape[0] <= m.shape[1] else m.t() @ m
                return float(t.linalg.eigvalsh(g)[-1].clamp_min(0).sqrt().item())
            if code == 0:
                out[q] = spec(f)
            elif code == 1:
                out[q] = spec(f) ** 2
            else:
                out[q] = max(spec(f[:rf2]) ** 2, spec(f[rf2:]))
        return out

    def _count(self, views):
        """nnz_factor: nonzeros of every payload window, counted on the device."""
        t = self.t
        if views.shape[0] == 0:
            return 0
        # column pieces of <= 65536 entries (dense_small.cu count_pieces_kernel);
        # the kernel resolves the pool / factor-buffer offsets itself
        views = np.ascontiguousarray(views, dtype=np.int64)
        cpp = np.maximum(1, 65536 // np.maximum(views[:, 2], 1))
        pstart = np.zeros(views.shape[0] + 1, dtype=np.int64)
        np.cumsum(np.where(views[:, 2] > 0, -(-views[:, 3] // cpp), 0), out=pstart[1:])
        if pstart[-1] == 0:
            return 0
        vd = to_dev(views)
        pd = to_dev(pstart)
        out = t.zeros(1, dtype=t.int64, device=dev())
        _lib.call("spand_count_nonzero_pieces", views.shape[0], ptr(vd), ptr(pd),
                  int(pstart[-1]), self.pool.data_ptr(), self.facbuf.data_ptr(), ptr(out),
                  stream())
        return int(out.item())


class LazyOps(Sequence):
    """The factor's operator list, built on access from the native
    collector's tables (the device apply and nnz never need the Python
    objects; tests, save_factor and user code get them on demand)."""

    def __init__(self, col, dofs, pool, fac):
        self.col, self.dofs, self.pool, self.fac = col, dofs, pool, fac
        self._rows = col.ops
        self._cache = {}
        self._perm_c = None

    def __len__(self):
        return self._rows.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        op = self._cache.get(i)
        if op is None:
            op = self._cache[i] = self._build(i)
        return op

    def _build(self, i):
        kind, c, li, wv, doff, size, _, lo, ld, linv, qo, rot, sb, se, lo_fac, _ = \
            self._rows[i].tolist()
        dofs, pool, fac, segs = self.dofs, self.pool, self.fac, self.col.segs
        if kind == 0:
            srows = segs[sb:se]
            return Elimination(dofs[c][doff:doff + size], _wd(dofs, srows),
                               MatView(pool, lo, ld, size, size), _pv(pool, srows, 0),
                               linv=MatView(fac, linv, ld, size, size))
        if kind == 1:
            return Scaling(dofs[c][doff:doff + size], MatView(fac, lo, ld, size, size),
                           linv=MatView(fac, linv, ld, size, size))
        if kind == 2:
            return Orthogonal(dofs[c][doff:doff + size],
                              MatView(fac, qo, max(ld, 1), size, size, rot=rot))
        if kind == 3:
            srows = segs[sb:se]
            return ErrorCorrection(dofs[c][doff:doff + size], _wd(dofs, srows),
                                   _pv(pool, srows, 1))
        if self._perm_c is None:
            self._perm_c = np.concatenate(dofs) if dofs else np.empty(0, np.int64)
        return Elimination(self._perm_c[self.col.fidx], np.empty(0, np.int64),
                           MatView(fac, lo, ld, size, size), [],
                           linv=MatView(fac, linv, ld, size, size))


def _wd(dofs, srows):
    """Lazy w_dofs: the neighbours' live dofs at the operator's time."""
    def build():
        if len(srows) == 0:
            return np.empty(0, np.int64)
        return np.concatenate([dofs[int(w)][int(wo):int(wo) + int(lw)]
                               for w, wo, lw in srows[:, :3]])
    return build


def _pv(pool, srows, axis):
    """Lazy payload views of a segment table: (MatView, offset) pairs stacked
    along rows (panels, axis 0) or columns (corrections, axis 1)."""
    def build():
        out, acc = [], 0
        for w, wo, lw, a, ld, r, c, tr in srows.tolist():
            out.append((MatView(pool, a, ld, r, c, bool(tr)), acc))
            acc += lw
        return out
    return build


class Collected:
    """Arrays of the native collector plus its handle (kept for the apply)."""

    def __init__(self, lib, h, vp):
        self.lib, self.h, self.vp = lib, h, vp
        sz = np.zeros(8, dtype=np.int64)
        lib.spand_collect_sizes(h, vp(sz))
        nops, nsegs, nperm, ndiag, nlsum, nviews, self.final_total, self.nfine = \
            (int(x) for x in sz)
        self.ops = np.zeros((nops, 16), dtype=np.int64)
        self.segs = np.zeros((nsegs, 8), dtype=np.int64)
        self.perm = np.zeros(nperm, dtype=np.int64)
        self.diag = np.zeros((ndiag, 10), dtype=np.int64)
        self.lsum = np.zeros((nlsum, 4), dtype=np.int64)
        self.views = np.zeros((nviews, 4), dtype=np.int64)
        self.fidx = np.zeros(self.final_total, dtype=np.int64)
        lib.spand_collect_get(h, vp(self.ops), vp(self.segs), vp(self.perm), vp(self.diag),
                              vp(self.lsum), vp(self.views), vp(self.fidx))

    def __del__(self):
        try:
            self.lib.spand_collect_destroy(self.h)
        except Exception:
            pass


def ctypes_ptr(addr):
    import ctypes
    return ctypes.c_void_p(int(addr))


def check_panel_rows(h, skip_levels):
    """Every cluster of depth d < levels - skip is sparsified at least once
    (levels d+1 .. levels-skip); its height must fit the device RRQR.
    Raises PanelTooLarge before anything is allocated or launched."""
    m0 = np.array([c.dofs.size for c in h.clusters], dtype=np.int64)
    dep = np.array([c.depth for c in h.clusters], dtype=np.int64)
    big = np.flatnonzero((dep < h.levels - skip_levels) & (m0 > MAX_PANEL_ROWS))
    if big.size:
        from .errors import PanelTooLarge
        c = int(big[np.argmax(m0[big])])
        raise PanelTooLarge(m0[c], MAX_PANEL_ROWS, cluster=h.clusters[c].id)


def run_factorization(a, h, eps, scheme, skip_levels, collect_local_errors=False,
                      near_kernel=None, digest=False):
    from .factorize import Factorization
    from .device import nvtx
    t0 = time.perf_counter()
    with nvtx("spand.symbolic"):
        eng = Engine(a, h, eps, scheme, skip_levels, near_kernel, collect_local_errors,
                     digest=digest)
    with nvtx("spand.factor_program"):
        eng.run()
    with nvtx("spand.collect"):
        ops, perm, diag, nnz = eng.collect()
    eng.timings["total_s"] = time.perf_counter() - t0
    f = Factorization(ops=ops, perm=perm, n=a.n, eps=float(eps), scheme=scheme,
                      skip_levels=int(skip_levels), nnz_factor=int(nnz),
                      diagnostics=diag,
                      _keep=(eng.pool, eng.facbuf, eng.geo), timings=eng.timings)
    f._plan = eng.apply_plan
    return f
