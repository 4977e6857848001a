"""collect_local_errors=True (reference factorize.py:296-339,
schemes.py:297-306,321-340): every sparsified interface records the spectral
norm of the term its sparsification drops.

Pinned against the reference's own values (tests/golden/local_errors.json,
``make_golden.py local_errors``): the oracle within 1e-12 relative, the
device path within 1e-8 relative (norms of the Q_f^T W rows the RRQR keeps
in the dead slots, computed on the device)."""

import json
import os

import numpy as np
import pytest

import paper_2007_00789_b200 as sp
from oracle import spand_oracle as orc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "local_errors.json")


def _cases():
    with open(GOLD) as fh:
        return json.load(fh)


def _parse(tag):
    _, d, lv, e, k, scheme = tag.split("_", 5)
    return int(d[1:]), int(lv[1:]), float(e[1:]), int(k[1:]), scheme


def _close(got, want, rtol):
    for (c1, v1), (c2, v2) in zip(got, want):
        assert c1 == c2
        assert abs(v1 - v2) <= rtol * max(abs(v2), 1e-300) + 1e-14, (c1, v1, v2)


@pytest.mark.parametrize("tag", sorted(_cases()))
def test_oracle_local_errors_match_reference(tag):
    want = _cases()[tag]
    d, lv, eps, skip, scheme = _parse(tag)
    a = sp.laplacian_2d(d)
    cl = orc.nd_hierarchy(a.n, a.row_ptr, a.col_idx, lv)
    f = orc.factorize(a.n, a.row_ptr, a.col_idx, a.values, cl, lv, eps, scheme, skip,
                      collect_local_errors=True)
    faces = [e[0] for lvd in f.diagnostics["levels"] for e in lvd["interfaces"]]
    got = list(zip(faces, f.diagnostics["local_errors"]))
    assert len(got) == len(want)
    _close(got, want, 1e-12)
    assert any(v > 0 for _, v in want)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(_cases()))
def test_device_local_errors_match_reference(tag):
    want = _cases()[tag]
    d, lv, eps, skip, scheme = _parse(tag)
    a = sp.laplacian_2d(d)
    h = sp.build_hierarchy(a, lv)
    f = sp.factorize(a, h, eps, scheme, skip_levels=skip, collect_local_errors=True)
    got = [[e["cluster"], e["local_error"]] for lvd in f.diagnostics["levels"]
           for e in lvd["interfaces"]]
    assert len(got) == len(want)
    _close(got, want, 1e-8)
    # the default path records none (and keeps only the correction rows)
    g = sp.factorize(a, h, eps, scheme, skip_levels=skip)
    assert all("local_error" not in e for lvd in g.diagnostics["levels"]
               for e in lvd["interfaces"])
