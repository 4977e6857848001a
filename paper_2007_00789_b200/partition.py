"""Nested-dissection hierarchy (host-side integer structure).

API of the reference `/root/reference/pkg/src/spdkit/partition.py:27-268`
(``Cluster``, ``PartitionHierarchy``, ``default_levels``, ``build_hierarchy``).
The recursion itself runs natively (``spand_nd_partition`` in
``csrc/partition.cpp``), restating the reference's BFS level-set bisection
bit for bit; ``tests/test_partition.py`` checks cluster lists against the
golden fixtures of the reference and the oracle.
"""

import ctypes
import json
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch


@dataclass(frozen=True)
class Cluster:
    """Unknowns handled as one unit; ``depth == levels`` marks leaves."""

    id: int
    dofs: np.ndarray
    depth: int

    @property
    def size(self):
        return len(self.dofs)


class PartitionHierarchy:
    """Interior/interface structure across levels (reference `:44-115`).

    At level l the interiors are the clusters of depth l and the interfaces
    the clusters of depth < l.
    """

    def __init__(self, levels, n, clusters, adj_ptr, adj_idx):
        self.levels = levels
        self.n = n
        self.clusters = clusters
        self._adj_ptr = adj_ptr
        self._adj_idx = adj_idx
        cluster_of = np.full(n, -1, dtype=np.int64)
        for c in clusters:
            cluster_of[c.dofs] = c.id
        self.cluster_of = cluster_of

    def interiors(self, level):
        return [c for c in self.clusters if c.depth == level]

    def interfaces(self, level):
        return [c for c in self.clusters if c.depth < level]

    def active(self, level):
        return [c for c in self.clusters if c.depth <= level]

    def promotion(self, level):
        """Level-l interfaces map to themselves at level l-1."""
        return {c.id: c.id for c in self.interfaces(level)}

    def neighbor_ids(self, cluster, level):
        active = {c.id for c in self.active(level)}
        out = set()
        for v in cluster.dofs:
            for w in self._adj_idx[self._adj_ptr[v]:self._adj_ptr[v + 1]]:
                cid = int(self.cluster_of[w])
                if cid != cluster.id and cid in active:
                    out.add(cid)
        return sorted(out)

    def level_view(self, level):
        out = []
        for c in self.active(level):
            out.append({
                "id": c.id,
                "kind": "interior" if c.depth == level else "interface",
                "dofs": [int(v) for v in c.dofs],
                "neighbors": self.neighbor_ids(c, level),
            })
        return out

    def to_json(self, path=None):
        doc = {
            "levels": self.levels,
            "n": self.n,
            "clusters": [{"id": c.id, "depth": c.depth,
                          "dofs": [int(v) for v in c.dofs]}
                         for c in self.clusters],
            "promotion": {str(l): self.promotion(l)
                          for l in range(1, self.levels + 1)},
        }
        if path is not None:
            with open(path, "w") as fh:
                json.dump(doc, fh)
        return doc


def default_levels(n):
    """Closest integer to log2(n/25), at least 1 (reference `:118-122`)."""
    if n < 2:
        raise ValueError("need at least 2 unknowns")
    return max(1, math.floor(math.log2(n / 25.0) + 0.5))


def _adjacency(a):
    rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.row_ptr))
    keep = rows != a.col_idx
    ptr = np.zeros(a.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=a.n), out=ptr[1:])
    return ptr, np.ascontiguousarray(a.col_idx[keep], dtype=np.int64)


def node_graph(a, block):
    """CSR pattern (row_ptr, col_idx, int64) of the graph whose vertices are
    the dof blocks {block*v, ..., block*v + block - 1} (e.g. the 3 dofs of an
    elasticity node): v ~ w iff any of their dofs are coupled in A."""
    if a.n % block:
        raise DimensionMismatch(f"n = {a.n} is not a multiple of block = {block}")
    nv = a.n // block
    rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.row_ptr)) // block
    cols = np.asarray(a.col_idx, dtype=np.int64) // block
    key = np.unique(rows * nv + cols)
    r, c = key // nv, key % nv
    ptr = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=nv), out=ptr[1:])
    return nv, ptr, np.ascontiguousarray(c, dtype=np.int64)


def build_hierarchy(a, levels, block=1):
    """Recursive vertex-separator dissection of the graph of A (native).

    ``block`` > 1 (EXTENSION for BASELINE config C5, not in the reference):
    dissect the graph of dof blocks (``node_graph``) with the same
    bisection, then expand every vertex to its ``block`` consecutive dofs, so
    the dofs of one node always share a cluster."""
    if block > 1:
        nv, rp, ci = node_graph(a, block)
        hn = _dissect(nv, rp, ci, levels)
        clusters = [Cluster(id=c.id, dofs=(block * c.dofs[:, None] +
                                            np.arange(block)).ravel(), depth=c.depth)
                    for c in hn]
        adj_ptr, adj_idx = _adjacency(a)
        return PartitionHierarchy(int(levels), int(a.n), clusters, adj_ptr, adj_idx)
    clusters = _dissect(int(a.n), a.row_ptr, a.col_idx, levels)
    adj_ptr, adj_idx = _adjacency(a)
    return PartitionHierarchy(int(levels), int(a.n), clusters, adj_ptr, adj_idx)


def _dissect(n, row_ptr, col_idx, levels):
    n = int(n)
    levels = int(levels)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    dofs = np.empty(n, dtype=np.int64)
    cptr = np.empty(n + 1, dtype=np.int64)
    depth = np.empty(max(n, 1), dtype=np.int32)
    ncl = np.zeros(1, dtype=np.int64)
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.call("spand_nd_partition", n, p(rp), p(ci), levels, p(dofs), p(cptr),
              p(depth), p(ncl))
    k = int(ncl[0])
    return [Cluster(id=i, dofs=dofs[cptr[i]:cptr[i + 1]].copy(), depth=int(depth[i]))
            for i in range(k)]
