"""Rebuild the inputs of the fixtures frozen by tests/golden/make_golden.py."""

import glob
import json
import os

import numpy as np

from paper_2007_00789_b200 import sparse as gen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(tag):
    with open(os.path.join(GOLDEN, tag + ".json")) as fh:
        rec = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, tag + ".npz")))
    return rec, arrays


def matrix_for(tag):
    """Same construction make_golden.py used for ``tag``."""
    if tag.startswith("lap2d_d"):
        d = int(tag.split("_")[1][1:])
        return gen.laplacian_2d(d)
    if tag.startswith("lap3d_d"):
        d = int(tag.split("_")[1][1:])
        return gen.laplacian_3d(d)
    if tag.startswith("hc2d_d64"):
        r = np.random.default_rng(2)
        return gen.diffusion_fv(gen.log_uniform_block_field((64, 64), 8, 3.0, r))
    if tag.startswith("hc3d_d16"):
        r = np.random.default_rng(3)
        return gen.diffusion_fv(
            gen.log_uniform_block_field((16, 16, 16), 4, 3.0, r))
    if tag.startswith("C5_ne"):
        return gen.c5_problem(int(tag.split("_")[1][2:]))[0]
    name = tag.split("_")[0]
    return gen.baseline_problem(name)[0]


def hierarchy_for(tag, a, levels):
    """The hierarchy make_golden.py handed to the reference: node-blocked
    (3 dofs per node) for the C5 elasticity cases, plain ND otherwise."""
    from paper_2007_00789_b200.partition import build_hierarchy
    return build_hierarchy(a, levels, block=3 if tag.startswith("C5") else 1)


def small_tags():
    tags = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        tag = os.path.basename(p)[:-5]
        if tag.startswith(("lap2d", "lap3d", "hc2d", "hc3d", "C1_")):
            tags.append(tag)
    return tags


def config_tags():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "C[2-5]_*.json"))):
        out.append(os.path.basename(p)[:-5])
    return out
