"""Fast structured apply plan for factors built by the device engine.

Same device kernels and phase order as ``apply.py`` (the level / wave
schedule that reproduces the reference's sequential operator order,
`factorize.py:269-282`), but built in the CLUSTER-CONTIGUOUS numbering: the
engine stores cluster c's slots at ``cstart[c] + [off[c], m0[c])``, so every
operator's dofs and each neighbour segment of its w_dofs is a contiguous
range.  Inputs are read as contiguous slices of a plan-owned permuted
vector (no index arrays), task and tile arrays are generated with NumPy in
bulk (no per-tile Python), and the vector is permuted in/out once per call.
"""

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .device import dev, ptr, require_cuda, stream, to_dev, to_dev_async


def ctypes_ptr(addr):
    import ctypes
    return ctypes.c_void_p(int(addr))

TILE_OUT = 64
TILE_K = 2048


class _Phase:
    __slots__ = ("tasks", "outs", "modes")

    def __init__(self):
        self.tasks = []   # task rows (8 ints)
        self.outs = []    # output start (int) or index array
        self.modes = []


def _task(view, optrans, in_start, out, mode, xb, idx_in=None):
    trans = bool(view.trans) != bool(optrans)
    if idx_in is not None:
        row = [view.addr, view.ld, view.rows, view.cols, int(trans), view.rot, 0, idx_in]
    else:
        row = [view.addr, view.ld, view.rows, view.cols, int(trans), view.rot, 1,
               xb + 8 * int(in_start)]
    return row, out, mode


class FastPlan:
    """apply_m / apply_inv / apply_inv_t of an engine factor."""

    def __init__(self, n, perm_new_to_old, arecs, n_phases):
        t = require_cuda()
        self.n = int(n)
        self.perm = to_dev(np.asarray(perm_new_to_old, dtype=np.int32), np.int32)
        self.xbuf = t.zeros(max(self.n, 1), dtype=t.float64, device=dev())
        xb = self.xbuf.data_ptr()
        fwd = [_Phase() for _ in range(n_phases)]
        bwd = [_Phase() for _ in range(n_phases)]
        idx_keep = []
        for rec in arecs:
            kind, (pf, pb) = rec[0], rec[1]
            if kind == "G":
                _, _, s0, ns, linv, segs = rec
                ph = fwd[pf["T"]]
                for x in (_task(linv, False, s0, s0, 0, xb),):
                    ph.tasks.append(x[0]); ph.outs.append(x[1]); ph.modes.append(0)
                ph = fwd[pf["A"]]
                for w0, nw, v in segs:
                    row, _, _ = _task(v, False, s0, w0, 1, xb)
                    ph.tasks.append(row); ph.outs.append(w0); ph.modes.append(1)
                ph = bwd[pb["A"]]
                for w0, nw, v in segs:
                    row, _, _ = _task(v, True, w0, s0, 1, xb)
                    ph.tasks.append(row); ph.outs.append(s0); ph.modes.append(1)
                ph = bwd[pb["T"]]
                row, _, _ = _task(linv, True, s0, s0, 0, xb)
                ph.tasks.append(row); ph.outs.append(s0); ph.modes.append(0)
            elif kind == "D":
                _, _, p0, m, linv = rec
                row, _, _ = _task(linv, False, p0, p0, 0, xb)
                fwd[pf["T"]].tasks.append(row); fwd[pf["T"]].outs.append(p0)
                fwd[pf["T"]].modes.append(0)
                row, _, _ = _task(linv, True, p0, p0, 0, xb)
                bwd[pb["T"]].tasks.append(row); bwd[pb["T"]].outs.append(p0)
                bwd[pb["T"]].modes.append(0)
            elif kind == "Q":
                _, _, p0, m, q = rec
                if m == 0:
                    continue
                row, _, _ = _task(q, True, p0, p0, 0, xb)
                fwd[pf["T"]].tasks.append(row); fwd[pf["T"]].outs.append(p0)
                fwd[pf["T"]].modes.append(0)
                row, _, _ = _task(q, False, p0, p0, 0, xb)
                bwd[pb["T"]].tasks.append(row); bwd[pb["T"]].outs.append(p0)
                bwd[pb["T"]].modes.append(0)
            elif kind == "E":
                _, _, p0, ncorr, segs = rec
                for w0, nw, v in segs:
                    row, _, _ = _task(v, True, p0, w0, 1, xb)
                    fwd[pf["A"]].tasks.append(row); fwd[pf["A"]].outs.append(w0)
                    fwd[pf["A"]].modes.append(1)
                for w0, nw, v in segs:
                    row, _, _ = _task(v, False, w0, p0, 1, xb)
                    bwd[pb["A"]].tasks.append(row); bwd[pb["A"]].outs.append(p0)
                    bwd[pb["A"]].modes.append(1)
            else:   # final dense block: index-array input (several clusters)
                _, _, fidx, total, linv = rec
                idx = to_dev(np.asarray(fidx, dtype=np.int32), np.int32)
                idx_keep.append(idx)
                for ph, tr in ((fwd[pf["T"]], False), (bwd[pb["T"]], True)):
                    row, _, _ = _task(linv, tr, 0, fidx, 0, xb, idx_in=idx.data_ptr())
                    ph.tasks.append(row); ph.outs.append(fidx); ph.modes.append(0)
        self._idx_keep = idx_keep
        self.fwd = self._compile(fwd)
        self.bwd = self._compile(bwd)
        self.scratch_len = max([p[-1] for p in self.fwd + self.bwd] + [1])
        self.scratch = t.empty(self.scratch_len, dtype=t.float64, device=dev())
        self._graph = None

    @staticmethod
    def _compile(phases):
        out = []
        for ph in phases:
            if not ph.tasks:
                continue
            tk = np.asarray(ph.tasks, dtype=np.int64)
            trans = tk[:, 4]
            nout = np.where(trans == 0, tk[:, 2], tk[:, 3])
            nk = np.where(trans == 0, tk[:, 3], tk[:, 2])
            keep = nout > 0
            tk, nout, nk = tk[keep], nout[keep], nk[keep]
            outs = [o for o, k in zip(ph.outs, keep) if k]
            modes = np.asarray(ph.modes, dtype=np.int64)[keep]
            if tk.shape[0] == 0:
                continue
            nkt = np.maximum(1, -(-nk // TILE_K))
            not_ = -(-nout // TILE_OUT)
            span = nout * nkt                       # scratch entries per task
            base = np.concatenate([[0], np.cumsum(span)[:-1]])
            # tiles: task-major, then k-chunk, then 64-output chunk
            per = not_ * nkt
            tid = np.repeat(np.arange(tk.shape[0]), per)
            loc = np.arange(int(per.sum())) - np.repeat(np.cumsum(per) - per, per)
            kbi = loc // np.repeat(not_, per)
            obi = loc % np.repeat(not_, per)
            ob = obi * TILE_OUT
            oc = np.minimum(TILE_OUT, nout[tid] - ob)
            kb = kbi * TILE_K
            kc = np.clip(nk[tid] - kb, 0, TILE_K)
            off = base[tid] + kbi * nout[tid] + ob
            tiles = np.stack([tid, ob, oc, kb, kc, off, np.zeros_like(tid),
                              np.zeros_like(tid)], axis=1).astype(np.int64)
            # scatter entries: every (task, k-chunk, output) in task order
            tot = int(span.sum())
            etid = np.repeat(np.arange(tk.shape[0]), span)
            eloc = np.arange(tot) - np.repeat(base, span)
            o = eloc % np.repeat(nout, span)
            src = np.arange(tot, dtype=np.int64)
            dst = np.empty(tot, dtype=np.int64)
            starts = np.fromiter((x if type(x) is int else -1 for x in outs),
                                 dtype=np.int64, count=len(outs))
            scal = starts >= 0
            m_sc = scal[etid]
            dst[m_sc] = starts[etid[m_sc]] + o[m_sc]
            if not scal.all():
                for k in np.flatnonzero(~scal):
                    sel = etid == k
                    dst[sel] = np.asarray(outs[k], dtype=np.int64)[o[sel]]
            mode = modes[etid]
            order = np.argsort(dst, kind="stable")
            dst, src, mode = dst[order], src[order], mode[order]
            first = np.r_[True, dst[1:] != dst[:-1]]
            st = np.flatnonzero(first)
            ptrs = np.r_[st, dst.size].astype(np.int64)
            out.append((to_dev_async(tk), to_dev_async(tiles), tiles.shape[0],
                        to_dev_async(dst[st].astype(np.int64)), to_dev_async(mode[st]),
                        to_dev_async(ptrs), to_dev_async(src), int(st.size), tot))
        return out

    @property
    def launches(self):
        return 2 * (len(self.fwd) + len(self.bwd)) + 2

    def _run_pass(self, phases):
        st = stream()
        x = self.xbuf
        for tasks, tiles, ntile, dst, mode, ptrs, src, nout, _ in phases:
            _lib.call("spand_gemv_tiles", ntile, ptr(tiles), ptr(tasks), ptr(x),
                      self.n, ptr(self.scratch), self.scratch_len, 1, st)
            _lib.call("spand_apply_scatter", nout, ptr(dst), ptr(mode), ptr(ptrs),
                      ptr(src), ptr(x), self.n, ptr(self.scratch), self.scratch_len,
                      1, st)

    def _run1(self, xd, forward, backward):
        st = stream()
        _lib.call("spand_gather", self.n, ptr(self.perm), ptr(xd), ptr(self.xbuf), st)
        if forward:
            self._run_pass(self.fwd)
        if backward:
            self._run_pass(self.bwd)
        _lib.call("spand_scatter_perm", self.n, ptr(self.perm), ptr(self.xbuf),
                  ptr(xd), st)

    GRAPH_AFTER = 32   # eager applies before a CUDA graph is captured

    def run_graph(self, xd):
        """apply_m in place on a contiguous (n,) fp64 device vector.  The
        first GRAPH_AFTER applies launch eagerly (capturing and instantiating
        a graph of ~350 kernels costs more than a short PCG solve); a factor
        reused for many solves switches to one CUDA graph replay."""
        t = require_cuda()
        self._napply = getattr(self, "_napply", 0) + 1
        if self._graph is None and self._napply <= self.GRAPH_AFTER:
            self._run1(xd, True, True)
            return xd
        if self._graph is None:
            self._gio = t.zeros(self.n, dtype=t.float64, device=dev())
            side = t.cuda.Stream()
            side.wait_stream(t.cuda.current_stream())
            g = t.cuda.CUDAGraph()
            with t.cuda.graph(g, stream=side):
                self._run1(self._gio, True, True)
            t.cuda.current_stream().wait_stream(side)
            self._graph = g
        self._gio.copy_(xd)
        self._graph.replay()
        _lib.COUNTS["apply_graph_kernels"] = (_lib.COUNTS.get("apply_graph_kernels", 0)
                                              + self.launches)
        xd.copy_(self._gio)
        return xd

    def run(self, xd, forward=True, backward=True):
        """In place on a device tensor of shape (n,) or (n, k)."""
        if xd.dim() == 1:
            self._run1(xd, forward, backward)
            return xd
        cols = xd.t().contiguous()
        for j in range(cols.shape[0]):
            self._run1(cols[j], forward, backward)
        xd.copy_(cols.t())
        return xd


_COMPILER = ThreadPoolExecutor(1, thread_name_prefix="spand-apply-image")
_PINNED = [None]


def _pinned_image(n):
    """Grow-only pinned int64 buffer for the apply images (compile thread)."""
    t = require_cuda()
    buf = _PINNED[0]
    if buf is None or buf.numel() < n:
        buf = t.empty(max(n, 2 * (buf.numel() if buf is not None else 0)), dtype=t.int64,
                      pin_memory=True)
        _PINNED[0] = buf
    return buf[:n]


class NativeApplyPlan(FastPlan):
    """The same structured apply, with the task / tile / scatter image built
    by the native collector (csrc/collect.cpp) instead of NumPy."""

    # attributes available once the host-compiled image is uploaded
    _LAZY = frozenset(("fwd", "bwd", "scratch", "scratch_len", "image", "image_host",
                       "phase_table", "build_times"))

    def __init__(self, n, perm_new_to_old, collected, pool, fac):
        """Allocate the device vectors and start compiling the apply image on
        a host thread (ctypes releases the GIL): the compile overlaps the rest
        of the factorization's host work (diagnostics, nnz count); the image
        is uploaded at the first apply."""
        t = require_cuda()
        self._t0 = time.perf_counter()
        self.n = int(n)
        self.perm = to_dev(np.asarray(perm_new_to_old, dtype=np.int32), np.int32)
        # NVEC_MAX permuted vectors, column-major (leading dimension n): the
        # image addresses column 0, the kernels step by n per right-hand side
        self.xbuf = t.zeros(max(self.n, 1) * self.NVEC_MAX, dtype=t.float64, device=dev())
        self._fidx = to_dev(np.asarray(collected.fidx if collected.fidx.size else [0],
                                       dtype=np.int32), np.int32)
        self._graph = None
        self._collected = collected
        self._future = _COMPILER.submit(self._compile_image, collected, pool.data_ptr(),
                                        fac.data_ptr(), self.xbuf.data_ptr(),
                                        self._fidx.data_ptr())

    @staticmethod
    def _compile_image(collected, pool_base, fac_base, xbuf, fidx):
        import ctypes
        lib, vp = collected.lib, collected.vp
        t0 = time.perf_counter()
        out = np.zeros(4, dtype=np.int64)
        lib.spand_collect_apply.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4 + \
            [ctypes.c_void_p]
        rc = lib.spand_collect_apply(collected.h, pool_base, fac_base, xbuf, fidx, vp(out))
        if rc != 0:
            raise RuntimeError(f"apply image build failed ({rc}): an operator exceeds "
                               "the packed work-item limits")
        t1 = time.perf_counter()
        ilen, nfw, nbw, scratch_len = (int(x) for x in out)
        # the image is written straight into pinned memory (reused between
        # factorizations: the previous plan's upload completed before the
        # next factorization's collect, which synchronises)
        pinned = _pinned_image(max(ilen, 1))
        image = pinned.numpy()
        ph = np.zeros((nfw + nbw, 10), dtype=np.int64)
        lib.spand_collect_apply_get.argtypes = [ctypes.c_void_p] * 3
        lib.spand_collect_apply_get(collected.h, vp(image), vp(ph))
        return pinned, ph, nfw, scratch_len, (t1 - t0, time.perf_counter() - t1)

    def __getattr__(self, name):
        if name in NativeApplyPlan._LAZY:
            self._ensure()
            return object.__getattribute__(self, name)
        raise AttributeError(name)

    def _ensure(self):
        import ctypes
        if "fwd" in self.__dict__:
            return
        t = require_cuda()
        pinned, ph, nfw, scratch_len, (t_setup, t_image) = self._future.result()
        t0 = time.perf_counter()
        self.scratch_len = scratch_len
        self.image = t.empty(pinned.shape, dtype=t.int64, device=dev())
        self.image.copy_(pinned, non_blocking=True)
        image = pinned.numpy()
        self.image_host = image   # (overwritten by the next factorization's image)
        base = self.image.data_ptr()
        self.scratch = t.empty(max(scratch_len, 1), dtype=t.float64, device=dev())
        rows = []
        for r in ph.tolist():
            to, nt, tio, nitem, co, nch, cbo, grid, _, _ = r
            rows.append((ctypes.c_void_p(base + 8 * to), ctypes.c_void_p(base + 8 * tio),
                         nitem, ctypes.c_void_p(base + 8 * co), nch,
                         ctypes.c_void_p(base + 8 * cbo), grid))
        self.phase_table = ph
        self.build_times = {"setup_s": t_setup, "image_s": t_image,
                            "upload_s": time.perf_counter() - t0, "image_mb": image.nbytes / 1e6,
                            "since_factor_s": time.perf_counter() - self._t0}
        self.bwd = rows[nfw:]
        self.fwd = rows[:nfw]

    NVEC_MAX = 8   # right-hand sides per multi-vector pass

    def _run_pass(self, phases, nvec=1):
        st = stream()
        x = self.xbuf
        scr = self.scratch if nvec == 1 else self._scratch_multi
        for tasks, items, nitem, chunks, nch, contrib, grid in phases:
            _lib.call("spand_gemv_items", nitem, grid, items, tasks, ptr(x), self.n,
                      ptr(scr), self.scratch_len, nvec, st)
            _lib.call("spand_apply_runs", nch, chunks, contrib, ptr(x), self.n,
                      ptr(scr), self.scratch_len, nvec, st)

    def run(self, xd, forward=True, backward=True):
        """In place on a device tensor of shape (n,) or (n, k); column stacks
        go through the factor NVEC_MAX vectors at a time (each payload
        element is read once per group of up to 4: GEMM-like reuse)."""
        if xd.dim() == 1:
            self._run1(xd, forward, backward)
            return xd
        t = require_cuda()
        if getattr(self, "_scratch_multi", None) is None:
            self._scratch_multi = t.empty(max(self.scratch_len, 1) * self.NVEC_MAX,
                                          dtype=t.float64, device=dev())
        cols = xd.t().contiguous()          # (k, n): vector j contiguous
        st = stream()
        n = self.n
        for j0 in range(0, cols.shape[0], self.NVEC_MAX):
            nv = min(self.NVEC_MAX, cols.shape[0] - j0)
            for v in range(nv):
                _lib.call("spand_gather", n, ptr(self.perm), ptr(cols[j0 + v]),
                          ctypes_ptr(self.xbuf.data_ptr() + 8 * n * v), st)
            if forward:
                self._run_pass(self.fwd, nv)
            if backward:
                self._run_pass(self.bwd, nv)
            for v in range(nv):
                _lib.call("spand_scatter_perm", n, ptr(self.perm),
                          ctypes_ptr(self.xbuf.data_ptr() + 8 * n * v), ptr(cols[j0 + v]), st)
        xd.copy_(cols.t())
        return xd
