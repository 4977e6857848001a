"""Structured apply plan for factors built by the device engine.

Same phase order as ``apply.py`` (the level / wave schedule that reproduces
the reference's sequential operator order, `factorize.py:269-282`), but in
the CLUSTER-CONTIGUOUS numbering: the engine stores cluster c's slots at
``cstart[c] + [off[c], m0[c])``, so every operator's dofs and each neighbour
segment of its w_dofs is a contiguous range.  The task / work-item / run
image is compiled natively (csrc/collect.cpp) on a host thread; inputs are
contiguous slices of a plan-owned permuted vector, permuted in/out once per
call.
"""

import os as _os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .device import dev, ptr, require_cuda, stream, to_dev


def ctypes_ptr(addr):
    import ctypes
    return ctypes.c_void_p(int(addr))

class FastPlan:
    """Shared driver of a structured apply plan: permute in, forward and/or
    backward phases, permute out; eager launches or one CUDA graph."""

    @property
    def launches(self):
        if getattr(self, "flow", None) is not None:
            return 3   # gather, one dataflow kernel (after a counter memset), scatter
        if getattr(self, "PERSISTENT", False) and getattr(self, "_ph", None) is not None:
            return 4   # gather, one cooperative kernel per pass, scatter
        return 2 * (len(self.fwd) + len(self.bwd)) + 2

    def _run_flow(self, nvec, scratch=None, ldscr=None):
        fl = self.flow
        _lib.call("spand_apply_dataflow", fl["nunit"], ptr(fl["units"]), ptr(fl["deps"]),
                  fl["nctr"], ptr(fl["ctrs"]), ptr(fl["phases"]), ptr(self.image),
                  ptr(self.xbuf), self.n, ptr(scratch if scratch is not None else fl["scratch"]),
                  ldscr or fl["scratch_len"], nvec, stream())
        _lib.COUNTS["spand_apply_dataflow"] = (_lib.COUNTS.get("spand_apply_dataflow", 0)
                                               + (nvec + 3) // 4 + (1 if nvec % 4 == 3 else 0))

    def _run1(self, xd, forward, backward):
        st = stream()
        _lib.call("spand_gather", self.n, ptr(self.perm), ptr(xd), ptr(self.xbuf), st)
        if forward and backward and getattr(self, "flow", None) is not None:
            self._run_flow(1)
            _lib.call("spand_scatter_perm", self.n, ptr(self.perm), ptr(self.xbuf),
                      ptr(xd), st)
            return
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
        self._maybe_swap()
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

_COMPILER = ThreadPoolExecutor(1, thread_name_prefix="spand-apply-image")


def _pinned_image(n):
    """Pinned int64 staging buffer of ONE plan's apply image.

    Each plan owns its buffer until its upload has been issued: a factor
    whose first apply comes after another factorization must upload its
    own rows (absolute pointers into its own pool / factor buffer), never
    the image of a later factor.  torch's caching host allocator recycles
    the block once the plan is gone and the non-blocking upload that read
    it has completed, so repeated factorizations do not re-pin memory."""
    t = require_cuda()
    return t.empty(n, dtype=t.int64, pin_memory=True)


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
        # the first image keeps every panel row (fast to compile: the first
        # applies wait for it); the row-compressed image (nonzero-row bits of
        # the elimination panels, a device scan) compiles in the background
        # after the first apply and replaces it once ready
        self._pool, self._fac = pool, fac
        self._future = _COMPILER.submit(self._compile_image, collected, pool.data_ptr(),
                                        fac.data_ptr(), self.xbuf.data_ptr(),
                                        self._fidx.data_ptr())
        self._future2 = None

    @staticmethod
    def _row_bits(collected, pool):
        import ctypes
        t = require_cuda()
        lib, vp = collected.lib, collected.vp
        sz = np.zeros(2, dtype=np.int64)
        lib.spand_collect_flag_sizes.argtypes = [ctypes.c_void_p] * 2
        lib.spand_collect_flag_sizes(collected.h, vp(sz))
        npan, nwords = int(sz[0]), int(sz[1])
        if npan == 0:
            return None, None
        rows = np.zeros(5 * npan, dtype=np.int64)
        lib.spand_collect_flag_panels.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                                  ctypes.c_void_p]
        lib.spand_collect_flag_panels(collected.h, pool.data_ptr(), vp(rows))
        rd = to_dev(rows, np.int64)
        bd = t.empty(max(nwords, 1), dtype=t.int32, device=dev())
        _lib.call("spand_row_bits", npan, ptr(rd), ptr(bd), stream())
        host = t.empty(bd.shape, dtype=t.int32, pin_memory=True)
        host.copy_(bd, non_blocking=True)
        ev = t.cuda.Event()
        ev.record()
        return (host, rd, bd), ev

    @staticmethod
    def _compile_image(collected, pool_base, fac_base, xbuf, fidx, bits=None, ready=None):
        import ctypes
        lib, vp = collected.lib, collected.vp
        t0 = time.perf_counter()
        bptr = None
        if bits is not None:
            ready.synchronize()
            bptr = ctypes.c_void_p(bits[0].data_ptr())
        t_bits = time.perf_counter() - t0
        out = np.zeros(4, dtype=np.int64)
        lib.spand_collect_apply.argtypes = [ctypes.c_void_p] + [ctypes.c_int64] * 4 + \
            [ctypes.c_void_p, ctypes.c_void_p]
        rc = lib.spand_collect_apply(collected.h, pool_base, fac_base, xbuf, fidx, bptr,
                                     vp(out))
        if rc != 0:
            raise RuntimeError(f"apply image build failed ({rc}): an operator exceeds "
                               "the packed work-item limits")
        t1 = time.perf_counter()
        ilen, nfw, nbw, scratch_len = (int(x) for x in out)
        # the image is written straight into this plan's pinned buffer
        pinned = _pinned_image(max(ilen, 1))
        image = pinned.numpy()
        ph = np.zeros((nfw + nbw, 10), dtype=np.int64)
        lib.spand_collect_apply_get.argtypes = [ctypes.c_void_p] * 3
        lib.spand_collect_apply_get(collected.h, vp(image), vp(ph))
        # the dataflow schedule of apply_m (one launch for both passes)
        dsz = np.zeros(4, dtype=np.int64)
        lib.spand_collect_dataflow_sizes.argtypes = [ctypes.c_void_p] * 2
        lib.spand_collect_dataflow_sizes(collected.h, vp(dsz))
        nunit, ndep, nctr, dscr = (int(v) for v in dsz)
        units = np.zeros(8 * max(nunit, 1), dtype=np.int64)
        deps = np.zeros(2 * max(ndep, 1), dtype=np.int64)
        dph = np.zeros(8 * max(nfw + nbw, 1), dtype=np.int64)
        lib.spand_collect_dataflow.argtypes = [ctypes.c_void_p] * 4
        lib.spand_collect_dataflow(collected.h, vp(units), vp(deps), vp(dph))
        flow = (nunit, units, deps, nctr, dscr, dph)
        return pinned, ph, nfw, scratch_len, (t1 - t0, time.perf_counter() - t1, t_bits), flow

    def __getattr__(self, name):
        if name in NativeApplyPlan._LAZY:
            self._ensure()
            return object.__getattribute__(self, name)
        raise AttributeError(name)

    ROW_COMPRESS = _os.environ.get("SPAND_APPLY_ROWBITS", "1") != "0"
    PERSISTENT = _os.environ.get("SPAND_APPLY_PERSISTENT", "0") == "1"

    def _ensure(self):
        if "fwd" in self.__dict__:
            return
        self._install(self._future.result(), compressed=False)
        if self.ROW_COMPRESS:
            bits, ready = self._row_bits(self._collected, self._pool)
            if bits is not None:
                self._future2 = _COMPILER.submit(
                    self._compile_image, self._collected, self._pool.data_ptr(),
                    self._fac.data_ptr(), self.xbuf.data_ptr(), self._fidx.data_ptr(), bits,
                    ready)

    def _maybe_swap(self):
        """Install the row-compressed image once its background compile is
        done (between applies; both images give the same bits, collect.cpp
        compile_phase); a captured graph is dropped."""
        f2 = getattr(self, "_future2", None)
        if f2 is not None and f2.done():
            self._future2 = None
            self._install(f2.result(), compressed=True)
            self._graph = None
            self._scratch_multi = None

    def _install(self, result, compressed):
        import ctypes
        t = require_cuda()
        pinned, ph, nfw, scratch_len, (t_setup, t_image, t_bits), flow = result
        t0 = time.perf_counter()
        self.scratch_len = scratch_len
        self.image = t.empty(pinned.shape, dtype=t.int64, device=dev())
        self.image.copy_(pinned, non_blocking=True)
        image = pinned.numpy()
        self.image_host = image
        base = self.image.data_ptr()
        self.scratch = t.empty(max(scratch_len, 1), dtype=t.float64, device=dev())
        rows = []
        for r in ph.tolist():
            to, nt, tio, nitem, co, nch, cbo, grid, _, _ = r
            rows.append((ctypes.c_void_p(base + 8 * to), ctypes.c_void_p(base + 8 * tio),
                         nitem, ctypes.c_void_p(base + 8 * co), nch,
                         ctypes.c_void_p(base + 8 * cbo), grid))
        self.phase_table = ph
        # host phase tables of the two passes (spand_apply_pass) and their
        # device copies (spand_apply_pass_persistent)
        self._ph = (np.ascontiguousarray(ph[:nfw]), np.ascontiguousarray(ph[nfw:]))
        self._phd = (to_dev(self._ph[0].ravel() if nfw else np.zeros(1, np.int64), np.int64),
                     to_dev(self._ph[1].ravel() if len(ph) > nfw else np.zeros(1, np.int64),
                            np.int64))
        if getattr(self, "_bar", None) is None:
            self._bar = t.zeros(2, dtype=t.int32, device=dev())
        bt = {"setup_s": t_setup, "image_s": t_image, "bits_wait_s": t_bits,
              "upload_s": time.perf_counter() - t0, "image_mb": image.nbytes / 1e6,
              "since_factor_s": time.perf_counter() - self._t0, "row_compressed": compressed}
        if compressed:
            self.build_times["compressed"] = bt
        else:
            self.build_times = bt
        self.bwd = rows[nfw:]
        self.fwd = rows[:nfw]
        nunit, units, deps, nctr, dscr, dph = flow
        self.flow = None
        if nunit > 0 and _os.environ.get("SPAND_APPLY_DATAFLOW", "0") == "1":
            self.flow = {"nunit": nunit, "units": to_dev(units, np.int64),
                         "deps": to_dev(deps, np.int64), "nctr": nctr,
                         "ctrs": t.zeros(nctr, dtype=t.int64, device=dev()),
                         "phases": to_dev(dph, np.int64), "scratch_len": dscr,
                         "scratch": t.empty(dscr, dtype=t.float64, device=dev())}
            self.build_times["dataflow_units"] = nunit
            self.build_times["dataflow_deps"] = int(deps.size // 2)
            self.build_times["dataflow_scratch_mb"] = 8 * dscr / 1e6

    NVEC_MAX = 8   # right-hand sides per multi-vector pass

    def _run_pass(self, phases, nvec=1):
        st = stream()
        x = self.xbuf
        scr = self.scratch if nvec == 1 else self._scratch_multi
        tab = getattr(self, "_ph", None)
        if tab is not None and self.PERSISTENT:
            # the whole pass in ONE cooperative launch (grid barriers between
            # the phases' item and accumulation stages)
            fw = phases is self.fwd
            ph = tab[0] if fw else tab[1]
            _lib.call("spand_apply_pass_persistent", len(ph), ptr(self._phd[0 if fw else 1]),
                      ptr(self.image), ptr(x), self.n, ptr(scr), self.scratch_len, nvec,
                      ptr(self._bar), st)
            _lib.COUNTS["spand_apply_pass_persistent"] = (
                _lib.COUNTS.get("spand_apply_pass_persistent", 0) + (nvec + 3) // 4
                + (1 if nvec % 4 == 3 else 0))
            return
        if tab is not None:
            # the whole pass in one native call (launch cost ~2 us per kernel
            # instead of ~5 us through ctypes per call)
            ph = tab[0] if phases is self.fwd else tab[1]
            _lib.call("spand_apply_pass", len(ph), ph.ctypes.data, ptr(self.image), ptr(x),
                      self.n, ptr(scr), self.scratch_len, nvec, st)
            ngv = (nvec // 4) + ((nvec % 4) // 2) + (nvec % 2)   # gemv launches per phase
            _lib.COUNTS["spand_gemv_items"] = _lib.COUNTS.get("spand_gemv_items", 0) + ngv * len(ph)
            _lib.COUNTS["spand_apply_runs"] = _lib.COUNTS.get("spand_apply_runs", 0) + len(ph)
            return
        for tasks, items, nitem, chunks, nch, contrib, grid in phases:
            _lib.call("spand_gemv_items", nitem, grid, items, tasks, ptr(x), self.n,
                      ptr(scr), self.scratch_len, nvec, st)
            _lib.call("spand_apply_runs", nch, chunks, contrib, ptr(x), self.n,
                      ptr(scr), self.scratch_len, nvec, st)

    def run(self, xd, forward=True, backward=True):
        """In place on a device tensor of shape (n,) or (n, k); column stacks
        go through the factor NVEC_MAX vectors at a time (each payload
        element is read once per group of up to 4: GEMM-like reuse)."""
        self._maybe_swap()
        if xd.dim() == 1:
            self._run1(xd, forward, backward)
            return xd
        cols = xd.t().contiguous()          # (k, n): vector j contiguous
        self.run_rows(cols, forward, backward)
        xd.copy_(cols.t())
        return xd

    def run_rows(self, cols, forward=True, backward=True):
        """In place on a contiguous (k, n) device tensor whose ROWS are the
        vectors (the multi-RHS PCG keeps its vectors this way); every row is
        transformed bit for bit as by the single-vector apply."""
        self._maybe_swap()
        t = require_cuda()
        if getattr(self, "_scratch_multi", None) is None:
            self._scratch_multi = t.empty(max(self.scratch_len, 1) * self.NVEC_MAX,
                                          dtype=t.float64, device=dev())
        st = stream()
        n = self.n
        for j0 in range(0, cols.shape[0], self.NVEC_MAX):
            nv = min(self.NVEC_MAX, cols.shape[0] - j0)
            for v in range(nv):
                _lib.call("spand_gather", n, ptr(self.perm), ptr(cols[j0 + v]),
                          ctypes_ptr(self.xbuf.data_ptr() + 8 * n * v), st)
            if forward and backward and getattr(self, "flow", None) is not None:
                fl = self.flow
                if fl.get("scratch_multi") is None:
                    fl["scratch_multi"] = t.empty(fl["scratch_len"] * 4, dtype=t.float64,
                                                  device=dev())
                self._run_flow(nv, fl["scratch_multi"], fl["scratch_len"])
            else:
                if forward:
                    self._run_pass(self.fwd, nv)
                if backward:
                    self._run_pass(self.bwd, nv)
            for v in range(nv):
                _lib.call("spand_scatter_perm", n, ptr(self.perm),
                          ctypes_ptr(self.xbuf.data_ptr() + 8 * n * v), ptr(cols[j0 + v]), st)
        return cols
