"""CPU ORACLE — test infrastructure only, never the product path.

A NumPy/SciPy restatement of the reference spaND hot path (spdkit 0.1.0,
`/root/reference/pkg/src/spdkit/`).  Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline leg may import it, and there only as the
checker / the timed CPU baseline.  The package ``paper_2007_00789_b200`` never
imports it: its numerical path is the sm_100a extension and fails loudly when
that is missing.

Parity pin: ``tests/test_oracle_golden.py`` checks this module against
fixtures frozen from the unmodified reference (``tests/golden/make_golden.py``):
hierarchy arrays, interface ranks, perm, per-op payload sha256 (bitwise), n_cg
and residual histories.  It uses the same NumPy/LAPACK primitives in the same
order as the reference, so on the same numpy/scipy build it is bitwise equal.

Each function cites the reference lines it restates.
"""

import math
import time

import numpy as np
import scipy.sparse as sp
from scipy.linalg import lapack, solve_triangular
from scipy.sparse.csgraph import connected_components, dijkstra

FIRST, FULL, SUPERFINE = "first", "second-full", "second-superfine"
SCHEMES = (FIRST, FULL, SUPERFINE)


class OracleNotSPD(Exception):
    def __init__(self, pivot):
        super().__init__(f"not SPD at pivot {pivot}")
        self.pivot = int(pivot)


# ---------------------------------------------------------------------------
# nested-dissection hierarchy  (partition.py:118-268)


def default_levels(n):
    """round(log2(n/25)), at least 1 (partition.py:118-122)."""
    return max(1, math.floor(math.log2(n / 25.0) + 0.5))


def _adjacency(n, row_ptr, col_idx):
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    off = rows != col_idx
    return sp.csr_matrix((np.ones(int(off.sum())), (rows[off], col_idx[off])),
                         shape=(n, n))


def _induced(adj_ptr, adj_idx, verts, local):
    """Induced subgraph in local numbering (partition.py:143-156)."""
    nv = verts.size
    local[verts] = np.arange(nv)
    lens = adj_ptr[verts + 1] - adj_ptr[verts]
    gather = (np.repeat(adj_ptr[verts] - np.cumsum(lens) + lens, lens)
              + np.arange(int(lens.sum())))
    cols = local[adj_idx[gather]]
    rows = np.repeat(np.arange(nv), lens)
    keep = cols >= 0
    local[verts] = -1
    ptr = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=nv), out=ptr[1:])
    return ptr, cols[keep]


def _neighbors_of(ptr, idx, nodes):
    lens = ptr[nodes + 1] - ptr[nodes]
    gather = (np.repeat(ptr[nodes] - np.cumsum(lens) + lens, lens)
              + np.arange(int(lens.sum())))
    return idx[gather], lens


def _bisect(adj_ptr, adj_idx, verts, local):
    """Level-set bisection with a pseudo-peripheral seed
    (partition.py:158-228).  Returns (part1, part2, separator)."""
    none = np.empty(0, dtype=np.int64)
    nv = verts.size
    if nv < 2:
        return verts, none, none
    ptr, idx = _induced(adj_ptr, adj_idx, verts, local)
    g = sp.csr_matrix((np.ones(idx.size), idx, ptr), shape=(nv, nv))
    ncomp, lab = connected_components(g, directed=False)
    if ncomp > 1:
        # whole components, largest first (ties: smaller label), greedily to
        # the lighter side (partition.py:173-185)
        sizes = np.bincount(lab)
        side = np.zeros(ncomp, dtype=np.int8)
        w1 = w2 = 0
        for c in np.lexsort((np.arange(ncomp), -sizes)):
            if w1 <= w2:
                side[c], w1 = 1, w1 + sizes[c]
            else:
                side[c], w2 = 2, w2 + sizes[c]
        return verts[side[lab] == 1], verts[side[lab] == 2], none
    far = dijkstra(g, directed=False, unweighted=True, indices=0)
    seed = int(np.flatnonzero(far == far.max())[0])
    dist = dijkstra(g, directed=False, unweighted=True,
                    indices=seed).astype(np.int64)
    order = np.lexsort((np.arange(nv), dist))
    width = np.bincount(dist)
    cum = np.cumsum(width)
    if width.size == 1:
        return none, none, verts
    other = nv - cum[:-1] - width[1:]
    best = int(np.argmin(np.abs(cum[:-1] - other)))
    cut = int(cum[best])
    side1 = order[:cut]
    nxt = int(width[best + 1])
    short = (nv - nxt) // 2 - cut
    if short > 0 and nxt > 1:
        layer = np.sort(order[cut:cut + nxt])
        side1 = np.concatenate([side1, layer[:min(short, nxt - 1)]])
    tag = np.zeros(nv, dtype=np.int8)          # 0 part2, 1 part1, 3 sep
    tag[side1] = 1
    nb, _ = _neighbors_of(ptr, idx, side1)
    tag[nb[tag[nb] == 0]] = 3
    sep = np.flatnonzero(tag == 3)
    if np.any(tag == 0) and sep.size:
        nb, lens = _neighbors_of(ptr, idx, sep)
        owner = np.repeat(np.arange(sep.size), lens)
        touches = np.bincount(owner[tag[nb] == 0], minlength=sep.size)
        tag[sep[touches == 0]] = 1
    return verts[tag == 1], verts[tag == 0], verts[tag == 3]


def nd_hierarchy(n, row_ptr, col_idx, levels):
    """Recursive dissection; clusters in DFS preorder, separator before its
    two halves (partition.py:231-268).  Returns [(id, dofs, depth)]."""
    adj = _adjacency(n, np.asarray(row_ptr), np.asarray(col_idx))
    aptr = adj.indptr.astype(np.int64)
    aidx = adj.indices.astype(np.int64)
    local = np.full(n, -1, dtype=np.int64)
    out = []

    def visit(verts, depth):
        if verts.size == 0:
            return
        if depth == levels or verts.size < 6:
            out.append((len(out), verts, levels))
            return
        p1, p2, sep = _bisect(aptr, aidx, verts, local)
        if sep.size == 0 and (p1.size == 0 or p2.size == 0):
            out.append((len(out), verts, levels))
            return
        if sep.size:
            out.append((len(out), sep, depth))
        visit(p1, depth + 1)
        visit(p2, depth + 1)

    visit(np.arange(n, dtype=np.int64), 0)
    return out


# ---------------------------------------------------------------------------
# dense kernels  (dense.py:45-222)


def chol(a):
    if a.shape[0] == 0:
        return np.zeros((0, 0))
    c, info = lapack.dpotrf(a, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise OracleNotSPD(info - 1)
    return c


def trinv(l):
    if l.shape[0] == 0:
        return np.zeros((0, 0))
    inv, info = lapack.dtrtri(l, lower=1)
    if info != 0:
        raise ValueError("singular triangle")
    return inv


def rrqr(a, coarse_tol, stop_tol):
    """Column-pivoted Householder QR with strict relative early stop
    (dense.py:117-183).  Returns q, r, perm, pivots, k_stop, k_c."""
    m, n = a.shape
    r = a.copy()
    q = np.eye(m)
    perm = np.arange(n)
    kmax = min(m, n)
    piv = np.zeros(kmax)
    if kmax == 0:
        return q, r, perm, piv, 0, 0
    cur = np.einsum("ij,ij->j", r, r)          # running squared norms
    ref = cur.copy()                            # value at last exact refresh
    r11 = 0.0
    k = 0
    while k < kmax:
        j = k + int(np.argmax(cur[k:]))
        eta = float(np.linalg.norm(r[k:, j]))   # exact pivot norm
        cur[j] = ref[j] = eta * eta
        if k == 0:
            r11 = eta
            if r11 == 0.0:
                break
        if eta < stop_tol * r11:
            break
        if j != k:
            for arr in (perm, cur, ref):
                arr[[k, j]] = arr[[j, k]]
            r[:, [k, j]] = r[:, [j, k]]
        piv[k] = eta
        if eta > 0.0:
            col = r[k:, k]
            beta = -eta if col[0] >= 0.0 else eta
            v = col.copy()
            v[0] -= beta
            tau = 2.0 / (v @ v)
            if k + 1 < n:
                w = (r[k:, k + 1:].T @ v) * tau
                r[k:, k + 1:] -= np.outer(v, w)
            r[k, k] = beta
            r[k + 1:, k] = 0.0
            qv = q[:, k:] @ v
            q[:, k:] -= np.outer(qv, v) * tau
            if k + 1 < n:
                row = r[k, k + 1:]
                tail = cur[k + 1:]
                tail -= row * row
                np.maximum(tail, 0.0, out=tail)
                stale = np.flatnonzero(tail < 0.01 * ref[k + 1:])
                if stale.size:
                    cols = k + 1 + stale
                    fresh = np.einsum("ij,ij->j", r[k + 1:, cols],
                                      r[k + 1:, cols])
                    cur[cols] = fresh
                    ref[cols] = fresh
        k += 1
    below = np.flatnonzero(piv[:k] < coarse_tol * r11)
    k_c = int(below[0]) if below.size else k
    return q, r, perm, piv, k, k_c


def sparsify_panel(panel, eps, scheme):
    """rrqr_sparsify (dense.py:186-222): returns dict with q_c, q_f,
    r_coarse, e_tilde, rank_c, rank_f2, perm, k_stop."""
    a = np.array(panel, dtype=np.float64, copy=True)
    m, n = a.shape
    stop = eps * eps if scheme == SUPERFINE else eps
    q, r, perm, piv, k_stop, k_c = rrqr(a, eps, stop)
    back = np.empty(n, dtype=np.int64)
    back[perm] = np.arange(n)
    out = {"perm": perm, "k_stop": k_stop, "pivots": piv,
           "q_c": np.ascontiguousarray(q[:, :k_c]),
           "q_f": np.ascontiguousarray(q[:, k_c:]),
           "r_coarse": np.ascontiguousarray(r[:k_c, :][:, back]),
           "rank_c": k_c, "rank_f2": 0}
    if scheme == FIRST:
        out["e_tilde"] = np.zeros((0, n))
    elif scheme == FULL:
        out["e_tilde"] = np.ascontiguousarray(r[k_c:, :][:, back])
    else:
        out["e_tilde"] = np.ascontiguousarray(r[k_c:k_stop, :][:, back])
        out["rank_f2"] = k_stop - k_c
    return out


# ---------------------------------------------------------------------------
# near-kernel preservation (EXTENSION, not in the reference: SURVEY.md §8a-11;
# the paper names it as compatible future work).
# With no vectors every function below reduces to the reference path bitwise.

NK_RTOL = 1e-8


def nk_basis(u, rtol=NK_RTOL):
    """Column-pivoted Householder QR of the restricted near-kernel block
    ``u`` (m x k): reflectors (v_t on rows t.., tau_t), the rank r (stop when
    the largest remaining column tail is <= rtol x the largest column norm)
    and R_u = (H^T u)[:r] with H = H_0 ... H_{r-1}.  Reflector convention of
    the reference RRQR (dense.py:155-159): beta = -sign(x0) eta."""
    x = np.array(u, dtype=np.float64, copy=True)
    m, k = x.shape
    vs, taus = [], []
    if m == 0 or k == 0:
        return vs, taus, x[:0]
    nrm0 = float(np.sqrt(np.max(np.einsum("ij,ij->j", x, x))))
    used = np.zeros(k, dtype=bool)
    for t in range(min(m, k)):
        tails = np.einsum("ij,ij->j", x[t:], x[t:])
        tails[used] = -1.0
        c = int(np.argmax(tails))
        eta = float(np.sqrt(tails[c]))
        if nrm0 == 0.0 or eta <= rtol * nrm0:
            break
        col = x[t:, c]
        beta = -eta if col[0] >= 0.0 else eta
        v = col.copy()
        v[0] -= beta
        tau = 2.0 / (v @ v)
        x[t:, :] -= np.outer(v, tau * (v @ x[t:, :]))
        used[c] = True
        vs.append(v)
        taus.append(tau)
    return vs, taus, x[:len(vs)].copy()


def nk_reflect(vs, taus, a):
    """H^T a = H_{r-1} ... H_0 a (rows of a)."""
    y = np.array(a, dtype=np.float64, copy=True)
    for t, (v, tau) in enumerate(zip(vs, taus)):
        y[t:] -= np.outer(v, tau * (v @ y[t:]))
    return y


def nk_explicit(vs, taus, m):
    """H = H_0 ... H_{r-1} as an explicit m x m matrix."""
    h = np.eye(m)
    for t in range(len(vs) - 1, -1, -1):
        v, tau = vs[t], taus[t]
        h[t:] -= np.outer(v, tau * (v @ h[t:]))
    return h


def sparsify_panel_nk(panel, u, eps, scheme):
    """Sparsification that keeps span(u) (the interface's restricted
    near-kernel vectors, m x k) inside the coarse basis.

    With H from ``nk_basis`` (U = H[:, :r], U_perp = H[:, r:]) the RRQR runs
    on the deflated panel U_perp^T W; the coarse basis is [U_perp q2_c, U]
    and the fine basis U_perp q2_f, so q = [q_f, q_c] stays orthogonal and
    fine-first.  r_coarse gains the rows U^T W; e_tilde is the RRQR's
    (q2_f^T U_perp^T W).  Returns (res, r, R_u); r == 0 is the reference
    path exactly (``sparsify_panel``)."""
    m, n = panel.shape
    vs, taus, ru = nk_basis(u) if n else ([], [], np.zeros((0, u.shape[1])))
    r = len(vs)
    if r == 0:
        return sparsify_panel(panel, eps, scheme), 0, ru
    y = nk_reflect(vs, taus, panel)
    res = sparsify_panel(y[r:], eps, scheme)
    h = nk_explicit(vs, taus, m)
    hp, hu = h[:, r:], h[:, :r]
    res["q_f"] = np.ascontiguousarray(hp @ res["q_f"])
    res["q_c"] = np.ascontiguousarray(np.hstack([hp @ res["q_c"], hu]))
    res["r_coarse"] = np.ascontiguousarray(np.vstack([res["r_coarse"], y[:r]]))
    res["rank_c"] += r
    return res, r, ru


# ---------------------------------------------------------------------------
# operators  (schemes.py:78-196)


class Op:
    """kind in 'G' (elimination), 'D' (scaling), 'Q' (orthogonal),
    'E' (error correction).  Fields follow schemes.py."""

    def __init__(self, kind, dofs, w_dofs=None, lower=None, panel=None,
                 q=None, e_tilde=None):
        self.kind = kind
        self.dofs = np.asarray(dofs, dtype=np.int64)
        self.w_dofs = (np.empty(0, np.int64) if w_dofs is None
                       else np.asarray(w_dofs, dtype=np.int64))
        self.lower, self.panel, self.q, self.e_tilde = lower, panel, q, e_tilde
        self._inv = None

    @property
    def linv(self):
        if self._inv is None:
            self._inv = trinv(self.lower)
        return self._inv

    def fwd(self, x):
        """apply_inv (schemes.py:102-106,136-137,162-163,188-189)."""
        k = self.kind
        if k == "G":
            t = self.linv @ x[self.dofs]
            x[self.dofs] = t
            if self.w_dofs.size:
                x[self.w_dofs] -= self.panel @ t
        elif k == "D":
            x[self.dofs] = self.linv @ x[self.dofs]
        elif k == "Q":
            x[self.dofs] = self.q.T @ x[self.dofs]
        else:
            x[self.w_dofs] -= self.e_tilde.T @ x[self.dofs]

    def bwd(self, x):
        """apply_inv_t (schemes.py:108-112,139-140,165-166,191-192)."""
        k = self.kind
        if k == "G":
            v = x[self.dofs]
            if self.w_dofs.size:
                v = v - self.panel.T @ x[self.w_dofs]
            x[self.dofs] = self.linv.T @ v
        elif k == "D":
            x[self.dofs] = self.linv.T @ x[self.dofs]
        elif k == "Q":
            x[self.dofs] = self.q @ x[self.dofs]
        else:
            x[self.dofs] -= self.e_tilde @ x[self.w_dofs]

    @property
    def nnz(self):
        if self.kind == "G":
            return int(np.count_nonzero(self.lower) +
                       np.count_nonzero(self.panel))
        if self.kind == "D":
            return int(np.count_nonzero(self.lower))
        if self.kind == "Q":
            return int(np.count_nonzero(self.q))
        return int(np.count_nonzero(self.e_tilde))


class Factor:
    def __init__(self, ops, perm, n, diagnostics):
        self.ops, self.perm, self.n = ops, perm, n
        self.diagnostics = diagnostics
        self.nnz_factor = int(sum(op.nnz for op in ops))

    def apply_inv(self, x):
        y = np.array(x, dtype=np.float64, copy=True)
        for op in self.ops:
            op.fwd(y)
        return y

    def apply_inv_t(self, x):
        y = np.array(x, dtype=np.float64, copy=True)
        for op in reversed(self.ops):
            op.bwd(y)
        return y

    def apply_m(self, x):
        return self.apply_inv_t(self.apply_inv(x))


# ---------------------------------------------------------------------------
# factorization driver  (factorize.py:51-366)


class _Trailing:
    """Block-sparse trailing matrix keyed by (i, j), i <= j
    (factorize.py:51-239)."""

    def __init__(self, n, row_ptr, col_idx, values, clusters):
        self.dofs = {cid: np.asarray(d, dtype=np.int64)
                     for cid, d, _ in clusters}
        self.depth = {cid: dep for cid, _, dep in clusters}
        self.alive = set(self.dofs)
        self.adj = {cid: set() for cid in self.alive}
        self.nk = None          # near-kernel coordinates (extension), n x k
        self.local_errors = False
        owner = np.full(n, -1, dtype=np.int64)
        slot = np.empty(n, dtype=np.int64)
        for cid, d in self.dofs.items():
            owner[d] = cid
            slot[d] = np.arange(d.size)
        rows = np.repeat(np.arange(n), np.diff(row_ptr))
        ci, cj = owner[rows], owner[col_idx]
        up = ci <= cj
        rows, cols, vals = rows[up], np.asarray(col_idx)[up], values[up]
        ci, cj = ci[up], cj[up]
        ncl = len(clusters)
        key = ci * ncl + cj
        o = np.argsort(key, kind="stable")
        key, rows, cols, vals = key[o], rows[o], cols[o], vals[o]
        cuts = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
        ends = np.r_[cuts[1:], key.size]
        self.blk = {}
        for s0, s1 in zip(cuts, ends):
            i, j = divmod(int(key[s0]), ncl)
            b = np.zeros((self.dofs[i].size, self.dofs[j].size))
            b[slot[rows[s0:s1]], slot[cols[s0:s1]]] = vals[s0:s1]
            self.blk[(i, j)] = b
            if i != j:
                self.adj[i].add(j)
                self.adj[j].add(i)

    def get(self, i, j):
        return self.blk[(i, j)] if i <= j else self.blk[(j, i)].T

    def row(self, cid, nbrs):
        if not nbrs:
            return (np.zeros((self.dofs[cid].size, 0)), np.empty(0, np.int64),
                    np.zeros(1, np.int64))
        sizes = [self.dofs[w].size for w in nbrs]
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        return (np.hstack([self.get(cid, w) for w in nbrs]),
                np.concatenate([self.dofs[w] for w in nbrs]), offs)

    def put_row(self, cid, nbrs, offs, rows):
        for t, w in enumerate(nbrs):
            piece = rows[:, offs[t]:offs[t + 1]]
            if cid <= w:
                self.blk[(cid, w)] = np.ascontiguousarray(piece)
            else:
                self.blk[(w, cid)] = np.ascontiguousarray(piece.T)

    def drop(self, cid, nbrs):
        for w in nbrs:
            self.blk.pop((min(cid, w), max(cid, w)), None)
            self.adj[w].discard(cid)
        self.blk.pop((cid, cid), None)
        self.adj.pop(cid, None)
        self.alive.discard(cid)

    def eliminate(self, cid):
        """factorize.py:131-163 + schemes.py:199-221."""
        nbrs = sorted(self.adj[cid])
        a_ss = self.blk[(cid, cid)]
        ns = a_ss.shape[0]
        if nbrs:
            a_ws = np.vstack([self.get(w, cid) for w in nbrs])
            w_dofs = np.concatenate([self.dofs[w] for w in nbrs])
        else:
            a_ws = np.zeros((0, ns))
            w_dofs = np.empty(0, np.int64)
        lower = chol(a_ss)
        if a_ws.shape[0]:
            panel = solve_triangular(lower, a_ws.T, lower=True, trans=0,
                                     check_finite=False).T
        else:
            panel = np.zeros((0, ns))
        upd = panel @ panel.T
        offs = np.concatenate([[0], np.cumsum(
            [self.dofs[w].size for w in nbrs])]).astype(np.int64)
        for a_, wi in enumerate(nbrs):
            for b_ in range(a_, len(nbrs)):
                wj = nbrs[b_]
                sub = upd[offs[a_]:offs[a_ + 1], offs[b_]:offs[b_ + 1]]
                have = self.blk.get((wi, wj))
                if have is None:
                    self.blk[(wi, wj)] = -sub
                    if wi != wj:
                        self.adj[wi].add(wj)
                        self.adj[wj].add(wi)
                else:
                    have -= sub
        op = Op("G", self.dofs[cid], w_dofs, lower=lower, panel=panel)
        self.drop(cid, nbrs)
        return op

    def rescale(self, cid):
        """factorize.py:165-173 + schemes.py:224-236."""
        nbrs = sorted(self.adj[cid])
        panel, _, offs = self.row(cid, nbrs)
        lower = chol(self.blk[(cid, cid)])
        if self.nk is not None:
            # near-kernel coordinates follow the congruence: u_p <- Z_p^T u_p
            d = self.dofs[cid]
            self.nk[d] = lower.T @ self.nk[d]
        if panel.size:
            scaled = solve_triangular(lower, panel, lower=True, trans=0,
                                      check_finite=False)
        else:
            scaled = np.zeros(panel.shape)
        self.blk[(cid, cid)] = np.eye(self.dofs[cid].size)
        self.put_row(cid, nbrs, offs, scaled)
        return Op("D", self.dofs[cid], lower=lower)

    def sparsify(self, cid, eps, scheme):
        """factorize.py:175-196 + schemes.py:272-318."""
        nbrs = sorted(self.adj[cid])
        panel, w_dofs, offs = self.row(cid, nbrs)
        old = self.dofs[cid]
        m = old.size
        if self.nk is None:
            res = sparsify_panel(panel, eps, scheme)
        else:
            res, r, ru = sparsify_panel_nk(panel, self.nk[old], eps, scheme)
            if r:
                # new coordinates: 0 on every slot but the last r (= R_u)
                self.nk[old] = 0.0
                self.nk[old[m - r:]] = ru
        n_fine = m - res["rank_c"]
        if self.local_errors:
            res["local_error"] = local_error(panel, res, scheme)
        ops = [Op("Q", old, q=np.hstack([res["q_f"], res["q_c"]]))]
        ops[0].pivots = res["pivots"][:res["k_stop"]]   # test-side metadata
        ops[0].k_c = res["rank_c"]
        ops[0].n_cols = panel.shape[1]
        ncorr = res["e_tilde"].shape[0]
        if ncorr and res["e_tilde"].size:
            ops.append(Op("E", old[:ncorr], w_dofs, e_tilde=res["e_tilde"]))
        kept = old[n_fine:]
        self.dofs[cid] = kept
        if kept.size:
            self.blk[(cid, cid)] = np.eye(kept.size)
            self.put_row(cid, nbrs, offs, res["r_coarse"])
        else:
            self.drop(cid, nbrs)
        return ops, old[:n_fine], res

    def finish(self):
        """factorize.py:198-220."""
        rest = sorted(self.alive)
        sizes = [self.dofs[c].size for c in rest]
        total = int(sum(sizes))
        if total == 0:
            return None, np.empty(0, np.int64)
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        dense = np.zeros((total, total))
        for a_, ci in enumerate(rest):
            for b_ in range(a_, len(rest)):
                blk = self.blk.get((ci, rest[b_]))
                if blk is None:
                    continue
                dense[offs[a_]:offs[a_ + 1], offs[b_]:offs[b_ + 1]] = blk
                if b_ != a_:
                    dense[offs[b_]:offs[b_ + 1], offs[a_]:offs[a_ + 1]] = blk.T
        dofs = np.concatenate([self.dofs[c] for c in rest])
        op = Op("G", dofs, np.empty(0, np.int64), lower=chol(dense),
                panel=np.zeros((0, total)))
        for c in rest:
            self.drop(c, sorted(self.adj[c]))
        return op, dofs


def local_error(panel, res, scheme):
    """Spectral norm of the dropped term (schemes.py:297-306, 321-340):
    first order ||Q_f^T W||, full second order ||E||^2, superfine
    max(||E||^2, ||Q_f1^T W||) with Q_f1 = Q_f[:, rank_f2:]."""
    def spec(a):
        return 0.0 if min(a.shape) == 0 else float(np.linalg.norm(a, 2))
    if scheme == FIRST:
        return spec(res["q_f"].T @ panel) if res["q_f"].size else 0.0
    if scheme == FULL:
        return spec(res["e_tilde"]) ** 2
    q_f1 = res["q_f"][:, res["rank_f2"]:]
    e1 = spec(q_f1.T @ panel) if q_f1.size else 0.0
    return max(spec(res["e_tilde"]) ** 2, e1)


def factorize(n, row_ptr, col_idx, values, clusters, levels, eps, scheme,
              skip_levels=4, near_kernel=None, collect_local_errors=False):
    """Level loop L..1 (factorize.py:285-366).  ``clusters`` is the
    [(id, dofs, depth)] list of ``nd_hierarchy``.  ``near_kernel`` (n or
    n x k, EXTENSION) switches on ``sparsify_panel_nk``."""
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}")
    if not 0.0 <= eps <= 1.0:
        raise ValueError(f"eps must lie in [0, 1], got {eps}")
    if skip_levels < 0:
        raise ValueError("skip_levels must be nonnegative")
    st = _Trailing(n, np.asarray(row_ptr), np.asarray(col_idx),
                   np.asarray(values, dtype=np.float64), clusters)
    st.local_errors = bool(collect_local_errors)
    lerr = []
    if near_kernel is not None:
        nk = np.array(near_kernel, dtype=np.float64, copy=True)
        nk = nk.reshape(n, -1)
        st.nk = nk if nk.shape[1] else None
    ops, perm_parts, diag = [], [], []
    for level in range(levels, 0, -1):
        inner = sorted(c for c in st.alive if st.depth[c] == level)
        ndofs = 0
        for cid in inner:
            d = st.dofs[cid]
            ops.append(st.eliminate(cid))
            perm_parts.append(d)
            ndofs += d.size
        skipped = (levels - level) < skip_levels
        faces = []
        if not skipped:
            iface = sorted(st.alive)
            for cid in iface:
                ops.append(st.rescale(cid))
            for cid in iface:
                before = st.dofs[cid].size
                new_ops, fine, res = st.sparsify(cid, eps, scheme)
                ops.extend(new_ops)
                if fine.size:
                    perm_parts.append(fine)
                faces.append([int(cid), int(before), int(res["rank_c"]),
                              int(res["rank_f2"])])
                if collect_local_errors:
                    lerr.append(res["local_error"])
        diag.append({"level": level, "interior_clusters": len(inner),
                     "interior_dofs": int(ndofs), "skipped": bool(skipped),
                     "interfaces": faces})
    last, last_dofs = st.finish()
    if last is not None:
        ops.append(last)
        perm_parts.append(last_dofs)
    perm = (np.concatenate(perm_parts) if perm_parts
            else np.empty(0, np.int64))
    out = {"levels": diag, "final_block": int(last_dofs.size)}
    if collect_local_errors:
        out["local_errors"] = lerr
    return Factor(ops, perm, n, out)


# ---------------------------------------------------------------------------
# PCG  (krylov.py:73-137)


def csr_matvec(n, row_ptr, col_idx, values):
    mat = sp.csr_matrix((values, col_idx, row_ptr), shape=(n, n))
    return lambda v: mat @ v


def pcg(apply_a, b, apply_m, tol, maxit=None):
    """Zero initial guess, recursive residual, strict rel < tol; returns
    (x, n_cg, history, converged, true_residual, seconds)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    if maxit is None:
        maxit = int(10.0 * math.sqrt(n) + 100.0)
    t0 = time.perf_counter()
    x = np.zeros(n)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return x, 0, [0.0], True, 0.0, time.perf_counter() - t0
    r = b.copy()
    hist = [1.0]
    z = apply_m(r)
    rz = float(r @ z)
    if rz <= 0.0:
        raise ArithmeticError("preconditioner not positive definite")
    p = z.copy()
    done = False
    its = 0
    for k in range(1, maxit + 1):
        ap = apply_a(p)
        pap = float(p @ ap)
        if pap <= 0.0:
            raise ArithmeticError("operator not positive definite")
        alpha = rz / pap
        x += alpha * p
        r -= alpha * ap
        rel = float(np.linalg.norm(r)) / bn
        hist.append(rel)
        its = k
        if rel < tol:
            done = True
            break
        z = apply_m(r)
        rz_new = float(r @ z)
        if rz_new <= 0.0:
            raise ArithmeticError("preconditioner not positive definite")
        p = z + (rz_new / rz) * p
        rz = rz_new
    true_res = float(np.linalg.norm(b - apply_a(x))) / bn
    return x, its, hist, done, true_res, time.perf_counter() - t0


# ---------------------------------------------------------------------------
# SPDF v1 factor container  (factorize.py:384-502)
#
# The checker's own reader/writer of the reference's byte format, so a
# factor written by the device path is read back by code that does not share
# anything with the product's reader (save_factor round trip, test_factorize.py
# :279-330).

SPDF_MAGIC = b"SPDF"
SPDF_HEADER = "<HqdBHIq"        # version, n, eps, scheme tag, skip, ops, nnz
SPDF_SCHEMES = {0: FIRST, 1: FULL, 2: SUPERFINE}
SPDF_KINDS = "GDQE"             # tags 0..3 (factorize.py:387-392)


class SPDFError(ValueError):
    pass


def _spdf_take(fh, count):
    data = fh.read(count)
    if len(data) != count:
        raise SPDFError("truncated factor file")
    return data


def _spdf_array(fh, dtype):
    import struct
    ndim = struct.unpack("<B", _spdf_take(fh, 1))[0]
    shape = struct.unpack(f"<{ndim}q", _spdf_take(fh, 8 * ndim))
    count = int(np.prod(shape)) if ndim else 1
    data = _spdf_take(fh, count * np.dtype(dtype).itemsize)
    return np.frombuffer(data, dtype=dtype).reshape(shape).copy()


def read_spdf(path):
    """load_factor (factorize.py:452-502) -> (Factor, header dict)."""
    import struct
    with open(path, "rb") as fh:
        if _spdf_take(fh, 4) != SPDF_MAGIC:
            raise SPDFError("not a factor file (bad magic)")
        ver, n, eps, stag, skip, nops, nnzf = struct.unpack(
            SPDF_HEADER, _spdf_take(fh, struct.calcsize(SPDF_HEADER)))
        if ver != 1:
            raise SPDFError(f"unsupported factor file version {ver}")
        if stag not in SPDF_SCHEMES:
            raise SPDFError(f"unknown scheme tag {stag}")
        perm = _spdf_array(fh, np.int64)
        ops = []
        for _ in range(nops):
            tag = struct.unpack("<B", _spdf_take(fh, 1))[0]
            if tag > 3:
                raise SPDFError(f"unknown operator tag {tag}")
            kind = SPDF_KINDS[tag]
            dofs = _spdf_array(fh, np.int64)
            if kind == "G":
                w = _spdf_array(fh, np.int64)
                low = _spdf_array(fh, np.float64)
                ops.append(Op("G", dofs, w, lower=low, panel=_spdf_array(fh, np.float64)))
            elif kind == "D":
                ops.append(Op("D", dofs, lower=_spdf_array(fh, np.float64)))
            elif kind == "Q":
                ops.append(Op("Q", dofs, q=_spdf_array(fh, np.float64)))
            else:
                w = _spdf_array(fh, np.int64)
                ops.append(Op("E", dofs, w, e_tilde=_spdf_array(fh, np.float64)))
    head = {"n": int(n), "eps": float(eps), "scheme": SPDF_SCHEMES[stag],
            "skip_levels": int(skip), "n_ops": int(nops), "nnz_factor": int(nnzf)}
    f = Factor(ops, perm, int(n), None)
    return f, head


def write_spdf(f, path, eps, scheme, skip_levels):
    """save_factor (factorize.py:424-449) for an oracle Factor."""
    import struct
    tag = {v: k for k, v in SPDF_SCHEMES.items()}[scheme]

    def put(fh, arr, dtype):
        arr = np.ascontiguousarray(arr, dtype=dtype)
        fh.write(struct.pack("<B", arr.ndim))
        fh.write(struct.pack(f"<{arr.ndim}q", *arr.shape))
        fh.write(arr.tobytes())

    with open(path, "wb") as fh:
        fh.write(SPDF_MAGIC)
        fh.write(struct.pack(SPDF_HEADER, 1, f.n, float(eps), tag, int(skip_levels),
                             len(f.ops), f.nnz_factor))
        put(fh, f.perm, np.int64)
        for op in f.ops:
            fh.write(struct.pack("<B", SPDF_KINDS.index(op.kind)))
            put(fh, op.dofs, np.int64)
            if op.kind == "G":
                put(fh, op.w_dofs, np.int64)
                put(fh, op.lower, np.float64)
                put(fh, op.panel, np.float64)
            elif op.kind == "D":
                put(fh, op.lower, np.float64)
            elif op.kind == "Q":
                put(fh, op.q, np.float64)
            else:
                put(fh, op.w_dofs, np.int64)
                put(fh, op.e_tilde, np.float64)


# ---------------------------------------------------------------------------
# Input generator of the BASELINE high-contrast configs (C3/C4 family), for
# the CPU legs of bench.py: the reference arm must not load the product, so
# its sample is built here.  Same construction as the package's
# sparse.diffusion_fv / log_uniform_block_field (cell-centred finite volumes,
# harmonic-mean faces, Dirichlet faces add the cell's own coefficient; the
# field is drawn first, then b); tests/test_host.py pins the two bitwise.


def fv_block_field_problem(shape, block, decades, seed):
    """(n, row_ptr, col_idx, values, b) of -div(a grad u) with a piecewise
    constant a = 10**U(-decades, decades) per block of block^d cells."""
    rng = np.random.default_rng(seed)
    nb = tuple(s // block for s in shape)
    a = 10.0 ** rng.uniform(-decades, decades, size=nb)
    for ax in range(len(shape)):
        a = np.repeat(a, block, axis=ax)
    n = a.size
    idx = np.arange(n).reshape(shape)
    diag = np.zeros(shape)
    rows, cols, vals = [], [], []
    for ax in range(a.ndim):
        lo = [slice(None)] * a.ndim
        hi = [slice(None)] * a.ndim
        lo[ax] = slice(0, shape[ax] - 1)
        hi[ax] = slice(1, shape[ax])
        a1, a2 = a[tuple(lo)], a[tuple(hi)]
        w = 2.0 * a1 * a2 / (a1 + a2)
        diag[tuple(lo)] += w
        diag[tuple(hi)] += w
        i0, i1 = idx[tuple(lo)].ravel(), idx[tuple(hi)].ravel()
        rows += [i0, i1]
        cols += [i1, i0]
        vals += [-w.ravel(), -w.ravel()]
        first = [slice(None)] * a.ndim
        last = [slice(None)] * a.ndim
        first[ax] = slice(0, 1)
        last[ax] = slice(shape[ax] - 1, shape[ax])
        diag[tuple(first)] += a[tuple(first)]
        diag[tuple(last)] += a[tuple(last)]
    rows.append(np.arange(n))
    cols.append(np.arange(n))
    vals.append(diag.ravel())
    m = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    m.sort_indices()
    b = rng.standard_normal(n)
    return (n, m.indptr.astype(np.int64), m.indices.astype(np.int64),
            m.data.astype(np.float64), b)


# ---------------------------------------------------------------------------
# Matrix Market reader  (sparse.py:98-160), the checker for csrc/mmio.cpp


class MMError(ValueError):
    """kind: 'ParseError' | 'NotSymmetricReal' | 'AsymmetricValues'."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def mm_read(path):
    """-> (n, row_ptr, col_idx, values) in CSR (both triangles, sorted)."""
    with open(path, "r") as fh:
        head = fh.readline()
        tok = head.strip().split()
        if len(tok) != 5 or tok[0] != "%%MatrixMarket":
            raise MMError("ParseError", f"bad Matrix Market header: {head.strip()!r}")
        if tok[1].lower() != "matrix" or tok[2].lower() != "coordinate":
            raise MMError("ParseError", f"unsupported object/format: {head.strip()!r}")
        if tok[3].lower() != "real" or tok[4].lower() != "symmetric":
            raise MMError("NotSymmetricReal", f"only real symmetric matrices are "
                          f"supported, got {tok[3]} {tok[4]}")
        line = fh.readline()
        while line and (line.startswith("%") or not line.strip()):
            line = fh.readline()
        try:
            m, n, nnz = (int(t) for t in line.split())
        except ValueError:
            raise MMError("ParseError", f"bad size line: {line.strip()!r}") from None
        if m != n:
            raise MMError("NotSymmetricReal", "matrix must be square")
        seen = {}
        for _ in range(nnz):
            line = fh.readline()
            if not line:
                raise MMError("ParseError", "file ends before declared entry count")
            t = line.split()
            if len(t) != 3:
                raise MMError("ParseError", f"bad entry line: {line.strip()!r}")
            try:
                i, j, v = int(t[0]), int(t[1]), float(t[2])
            except ValueError:
                raise MMError("ParseError", f"bad entry line: {line.strip()!r}") from None
            if not (1 <= i <= n and 1 <= j <= n):
                raise MMError("ParseError", f"index out of range: ({i}, {j})")
            if (i - 1, j - 1) in seen:
                raise MMError("ParseError", f"duplicate entry ({i}, {j})")
            mir = (j - 1, i - 1)
            if i != j and mir in seen and seen[mir] != v:
                raise MMError("AsymmetricValues", f"entries ({j}, {i}) and ({i}, {j}) "
                              f"disagree: {seen[mir]} vs {v}")
            seen[(i - 1, j - 1)] = v
    rows, cols, vals = [], [], []
    for (i, j), v in seen.items():
        rows.append(i)
        cols.append(j)
        vals.append(v)
        if i != j and (j, i) not in seen:
            rows.append(j)
            cols.append(i)
            vals.append(v)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rp[1:])
    return n, rp, cols[order], vals[order]
