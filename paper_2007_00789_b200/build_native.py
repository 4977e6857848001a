"""Build the sm_100a shared library ``libspand_b200.so`` in-tree.

    python -m paper_2007_00789_b200.build_native

One nvcc invocation per translation unit (``-gencode
arch=compute_100a,code=sm_100a -lineinfo -O3``), linked with ``-shared``.
The .so lands next to this file so it travels with the repo snapshot to the
GPU box; nothing is installed into site-packages.
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libspand_b200.so")
BUILD = os.path.join(HERE, "csrc", "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "nvcc")
PER_FILE = {}   # per-file extra nvcc flags


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(CSRC, "*.h")) + [os.path.join(HERE, "..", "include",
                                                    "spand_b200.h")]
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose=False, jobs=8):
    os.makedirs(BUILD, exist_ok=True)
    objs, procs = [], []
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if not _stale(obj, src):
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17",
               "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
               "-c", src, "-o", obj]
        if os.path.basename(src) in PER_FILE:
            cmd[1:1] = PER_FILE[os.path.basename(src)]
        if src.endswith(".cpp"):
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT)))
        if len(procs) >= jobs:
            _drain(procs, verbose)
    _drain(procs, verbose)
    if (not os.path.exists(OUT) or
            any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs)):
        cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return OUT


def _drain(procs, verbose):
    while procs:
        src, p = procs.pop(0)
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{text}")
        if verbose and text.strip():
            print(text)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
