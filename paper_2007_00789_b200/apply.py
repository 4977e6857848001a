"""Batched device apply of the factor: M x = L^-T (L^-1 x).

Replaces the reference's per-operator loop (`factorize.py:269-282`) and the
operator bodies (`schemes.py:102-112,136-140,162-166,188-192`).

Each operator splits into micro-ops of two shapes:
  T  (transform in place)   x[S] <- M x[S]            (reads S, overwrites S)
  A  (accumulate)           x[W] -= M x[R]            (reads R, subtracts into W)
forward:  G = T(Linv) then A(panel);  D = T(Linv);  Q = T(q^T);  E = A(e^T)
backward: G = A(panel^T) then T(Linv^T); D = T(Linv^T); Q = T(q); E = A(e)
(backward walks the operators in reverse order, `factorize.py:275-279`).

A greedy scheduler places every micro-op in the earliest PHASE that keeps
all read-after-write, write-after-read and write-after-write orders of the
sequential reference; accumulations into the same entry may share a phase
and are summed in sequence order.  A phase is two launches: one batched
GEMV over 64-output x 2048-inner tiles (spand_gemv_tiles) and one ordered
scatter (spand_apply_scatter).  The result is deterministic run to run.
"""

import numpy as np

from . import _lib
from .device import dev, ptr, require_cuda, stream, to_dev, to_dev_async
from .schemes import MatView, OpKind

TILE_OUT = 64
TILE_K = 2048


class _Micro:
    __slots__ = ("reads", "writes", "accs", "tasks", "mode", "phase")

    def __init__(self, reads, writes, accs, tasks, mode):
        self.reads, self.writes, self.accs = reads, writes, accs
        self.tasks = tasks        # [(MatView, optrans, in_dofs, out_dofs)]
        self.mode = mode          # 0 overwrite-with-sum, 1 subtract-sum
        self.phase = None         # structural phase (engine factors) or None


def _views(op):
    """(linv, panel views, q, e views) of an operator."""
    return (getattr(op, "linv_view", None), getattr(op, "panel_views", None),
            getattr(op, "q_view", None), getattr(op, "e_views", None))


def _micro_ops(op, backward):
    k = op.kind
    linv, pviews, qv, eviews = _views(op)
    s = op.dofs
    out = []
    if k is OpKind.ELIMINATION:
        w = op.w_dofs
        t_op = _Micro(s, s, None, [(linv, backward, s, s)], 0)
        a_tasks = []
        for v, r0 in (pviews or []):
            nr = v.shape[0]
            if nr == 0 or s.size == 0:
                continue
            wr = w[r0:r0 + nr]
            if backward:
                a_tasks.append((v, True, wr, s))
            else:
                a_tasks.append((v, False, s, wr))
        if backward:
            if a_tasks:
                out.append(_Micro(w, None, s, a_tasks, 1))
            out.append(t_op)
        else:
            out.append(t_op)
            if a_tasks:
                out.append(_Micro(s, None, w, a_tasks, 1))
    elif k is OpKind.SCALING:
        out.append(_Micro(s, s, None, [(linv, backward, s, s)], 0))
    elif k is OpKind.ORTHOGONAL:
        out.append(_Micro(s, s, None, [(qv, not backward, s, s)], 0))
    else:
        w = op.w_dofs
        tasks = []
        for v, c0 in (eviews or []):
            nc = v.shape[1]
            if nc == 0 or s.size == 0:
                continue
            wc = w[c0:c0 + nc]
            if backward:
                tasks.append((v, False, wc, s))
            else:
                tasks.append((v, True, s, wc))
        if tasks:
            if backward:
                out.append(_Micro(w, None, s, tasks, 1))
            else:
                out.append(_Micro(s, None, w, tasks, 1))
    # structural phases supplied by the engine: "T" (transform) and "A"
    # (accumulate) micro-ops of this operator in this direction
    ph = getattr(op, "_phases", None)
    if ph is not None:
        key = 1 if backward else 0
        for m in out:
            m.phase = ph[key]["T" if m.writes is not None else "A"]
    # drop empty transforms (0-sized blocks)
    return [m for m in out if m.tasks and (m.writes is None or m.writes.size)]


def _schedule(micro, n):
    """Earliest phase of every micro-op (see module docstring)."""
    lr = np.full(n, -1, dtype=np.int64)
    lw = np.full(n, -1, dtype=np.int64)
    la = np.full(n, -1, dtype=np.int64)
    phase = np.empty(len(micro), dtype=np.int64)
    for i, m in enumerate(micro):
        p = 0
        R, W, C = m.reads, m.writes, m.accs
        if R is not None and R.size:
            p = max(p, int(lw[R].max()) + 1, int(la[R].max()) + 1)
        if W is not None and W.size:
            p = max(p, int(lr[W].max()), int(lw[W].max()) + 1,
                    int(la[W].max()) + 1)
        if C is not None and C.size:
            p = max(p, int(lr[C].max()), int(lw[C].max()) + 1,
                    int(la[C].max()))
        phase[i] = p
        if R is not None and R.size:
            lr[R] = np.maximum(lr[R], p)
        if W is not None and W.size:
            lw[W] = np.maximum(lw[W], p)
        if C is not None and C.size:
            la[C] = np.maximum(la[C], p)
    return phase


class _Pass:
    """Device arrays of one direction (forward or backward)."""

    def __init__(self, n, micro, idx_pool):
        self.phases = []
        if not micro:
            self.scratch_len = 0
            return
        if all(m.phase is not None for m in micro):
            # engine factors: phases follow the level / wave structure
            # (same dependency order as the sequential reference, no search)
            ph = np.asarray([m.phase for m in micro], dtype=np.int64)
            uniq = np.unique(ph)
            ph = np.searchsorted(uniq, ph)
        else:
            ph = _schedule(micro, n)
        nph = int(ph.max()) + 1
        by_phase = [[] for _ in range(nph)]
        for i, p in enumerate(ph):
            by_phase[p].append(micro[i])
        task_rows, tile_lists, scat = [], [], []
        scratch_len = 0
        for plist in by_phase:
            tiles = []
            dst_parts, lens, modes = [], [], []
            pos = 0
            for m in plist:
                for (v, optrans, in_dofs, out_dofs) in m.tasks:
                    trans = bool(v.trans) != bool(optrans)
                    nout = v.cols if trans else v.rows
                    nk = v.rows if trans else v.cols
                    if nout == 0:
                        continue
                    tid = len(task_rows)
                    task_rows.append([v.addr, v.ld, v.rows, v.cols, int(trans),
                                      v.rot, 0, idx_pool.addr(in_dofs)])
                    nkt = max(1, -(-nk // TILE_K))
                    for ob in range(0, nout, TILE_OUT):
                        oc = min(TILE_OUT, nout - ob)
                        for kb in range(0, nkt * TILE_K, TILE_K):
                            tiles.append([tid, ob, oc, kb, min(TILE_K, nk - kb) if nk else 0,
                                          pos, 0, 0])
                            pos += oc
                    if nkt == 1:
                        dst_parts.append(out_dofs[:nout])
                    else:
                        dst_parts.append(np.concatenate(
                            [np.tile(out_dofs[ob:ob + TILE_OUT], nkt)
                             for ob in range(0, nout, TILE_OUT)]))
                    lens.append(nout * nkt)
                    modes.append(m.mode)
            scratch_len = max(scratch_len, pos)
            tile_lists.append(np.asarray(tiles, dtype=np.int64).reshape(-1, 8))
            if dst_parts:
                dst = np.concatenate(dst_parts)
                src = np.arange(dst.size, dtype=np.int64)   # tiles are laid out in order
                mode = np.repeat(np.asarray(modes, dtype=np.int64), lens)
                order = np.argsort(dst, kind="stable")      # keeps sequence order
                dst, src, mode = dst[order], src[order], mode[order]
                first = np.r_[True, dst[1:] != dst[:-1]]
                starts = np.flatnonzero(first)
                ptrs = np.r_[starts, dst.size].astype(np.int64)
                scat.append((dst[starts].astype(np.int64), mode[starts],
                             ptrs, src))
            else:
                scat.append(None)
        self.scratch_len = scratch_len
        self.tasks = to_dev_async(np.asarray(task_rows, dtype=np.int64).reshape(-1, 8))
        for tl, sc in zip(tile_lists, scat):
            if tl.shape[0] == 0:
                continue
            dst, mode, ptrs, src = sc
            self.phases.append((to_dev_async(tl), tl.shape[0], to_dev_async(dst),
                                to_dev_async(mode), to_dev_async(ptrs), to_dev_async(src),
                                dst.size))

    def run(self, x, scratch, ldx, ldscr, nvec):
        st = stream()
        for tiles, ntile, dst, mode, ptrs, src, nout in self.phases:
            _lib.call("spand_gemv_tiles", ntile, ptr(tiles), ptr(self.tasks),
                      ptr(x), ldx, ptr(scratch), ldscr, nvec, st)
            _lib.call("spand_apply_scatter", nout, ptr(dst), ptr(mode), ptr(ptrs),
                      ptr(src), ptr(x), ldx, ptr(scratch), ldscr, nvec, st)

    @property
    def launches(self):
        return 2 * len(self.phases)


class _IndexPool:
    """All gather index arrays of a plan in one device int32 buffer."""

    def __init__(self):
        self._parts, self._where, self._len = [], {}, 0
        self.buf = None

    def add(self, arr):
        key = (arr.__array_interface__["data"][0], arr.size,
               arr.strides[0] if arr.ndim else 0)
        if key not in self._where:
            self._where[key] = self._len
            self._parts.append(np.asarray(arr, dtype=np.int32))
            self._len += arr.size
        return self._where[key]

    def finish(self):
        data = (np.concatenate(self._parts) if self._parts
                else np.zeros(1, np.int32))
        self.buf = to_dev(data, np.int32)

    def addr(self, arr):
        key = (arr.__array_interface__["data"][0], arr.size,
               arr.strides[0] if arr.ndim else 0)
        return self.buf.data_ptr() + 4 * self._where[key]


class ApplyPlan:
    """Forward and backward device passes over a factor's operator list."""

    def __init__(self, n, ops):
        require_cuda()
        self.n = int(n)
        fwd, bwd = [], []
        for op in ops:
            fwd.extend(_micro_ops(op, backward=False))
        for op in reversed(ops):
            bwd.extend(_micro_ops(op, backward=True))
        pool = _IndexPool()
        for m in fwd + bwd:
            for (_, _, a, b) in m.tasks:
                pool.add(a)
        pool.finish()
        self._pool = pool
        self.fwd = _Pass(self.n, fwd, pool)
        self.bwd = _Pass(self.n, bwd, pool)
        self.scratch_len = max(self.fwd.scratch_len, self.bwd.scratch_len, 1)
        self._scratch = None
        self._graph = None

    @property
    def launches(self):
        return self.fwd.launches + self.bwd.launches

    def _scr(self, nvec):
        t = require_cuda()
        need = self.scratch_len * nvec
        if self._scratch is None or self._scratch.numel() < need:
            self._scratch = t.empty(need, dtype=t.float64, device=dev())
        return self._scratch

    def run_graph(self, xd):
        """apply_m in place on a contiguous (n,) fp64 device tensor through a
        CUDA graph of the whole pass (captured on first use: ~2 launches
        per phase collapse into one graph launch)."""
        t = require_cuda()
        if self._graph is None:
            self._xbuf = t.zeros(self.n, dtype=t.float64, device=dev())
            scr = self._scr(1)
            side = t.cuda.Stream()
            side.wait_stream(t.cuda.current_stream())
            g = t.cuda.CUDAGraph()
            with t.cuda.graph(g, stream=side):
                self.fwd.run(self._xbuf, scr, self.n, self.scratch_len, 1)
                self.bwd.run(self._xbuf, scr, self.n, self.scratch_len, 1)
            t.cuda.current_stream().wait_stream(side)
            self._graph = g
        self._xbuf.copy_(xd)
        self._graph.replay()
        _lib.COUNTS["apply_graph_kernels"] = (_lib.COUNTS.get("apply_graph_kernels", 0)
                                              + self.launches)
        xd.copy_(self._xbuf)
        return xd

    def run(self, xd, forward=True, backward=True):
        """In-place on a device tensor of shape (n,) or (n, k) (fp64)."""
        if xd.dim() == 1:
            xs, nvec = xd, 1
        else:
            xs, nvec = xd.t().contiguous(), xd.shape[1]
        scr = self._scr(nvec)
        if forward:
            self.fwd.run(xs, scr, self.n, self.scratch_len, nvec)
        if backward:
            self.bwd.run(xs, scr, self.n, self.scratch_len, nvec)
        if xd.dim() != 1:
            xd.copy_(xs.t())
        return xd


def apply_single(op, x, transpose):
    """Apply one operator in place to a NumPy vector/stack (device round
    trip; used only by callers that drive operators one at a time)."""
    t = require_cuda()
    n = x.shape[0]
    plan = ApplyPlan(n, [op])
    xd = t.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev())
    plan.run(xd, forward=not transpose, backward=transpose)
    x[...] = xd.cpu().numpy()
