"""ctypes binding of the C-ABI in include/spand_b200.h.

The library is REQUIRED: importing a numerical entry point without it (or
without a CUDA device) raises NativeUnavailable; there is no host fallback.
"""

import ctypes
import os

from .errors import NativeUnavailable

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPAND_LIB_PATH") or os.path.join(HERE, "libspand_b200.so")

_c_int, _c_dbl, _c_i64 = ctypes.c_int, ctypes.c_double, ctypes.c_int64
_P = ctypes.c_void_p

# name -> argtypes (all return int)
SIGNATURES = {
    "spand_version": [],
    "spand_device_sm_count": [],
    "spand_spmv_blocks": [_c_int],
    "spand_csr_spmv": [_c_int, _P, _P, _P, _P, _P, _P, _P],
    "spand_dot_blocks": [_c_int],
    "spand_dot": [_c_int, _P, _P, _P, _P, _P],
    "spand_reduce_sum": [_c_int, _P, _P, _P],
    "spand_pcg_xr": [_c_int, _P, _P, _P, _P, _P, _P, _P],
    "spand_pcg_p": [_c_int, _P, _P, _P, _P],
    "spand_gather": [_c_int, _P, _P, _P, _P],
    "spand_scatter_perm": [_c_int, _P, _P, _P, _P],
    "spand_gemv_tiles": [_c_int, _P, _P, _P, _c_i64, _P, _c_i64, _c_int, _P],
    "spand_gemv_items": [_c_int, _c_int, _P, _P, _P, _c_i64, _P, _c_i64, _c_int, _P],
    "spand_apply_scatter": [_c_int, _P, _P, _P, _P, _P, _c_i64, _P, _c_i64,
                            _c_int, _P],
    "spand_apply_runs": [_c_int, _P, _P, _P, _c_i64, _P, _c_i64, _c_int, _P],
    "spand_apply_pass": [_c_int, _P, _P, _P, _c_i64, _P, _c_i64, _c_int, _P],
    "spand_row_bits": [_c_int, _P, _P, _P],
    "spand_apply_pass_persistent": [_c_int, _P, _P, _P, _c_i64, _P, _c_i64, _c_int, _P, _P],
    "spand_run_launches": [_c_int, _P, _c_i64, _P, _P, _P, _P, _c_i64, _P, _c_dbl, _c_int, _P,
                           _c_i64, _c_int, _c_dbl, _c_int, _P, _P],
    "spand_launch_timer_reset": [],
    "spand_launch_timer_read": [_P, _P],
    "spand_apply_dataflow": [_c_i64, _P, _P, _c_i64, _P, _P, _P, _P, _c_i64, _P, _c_i64, _c_int,
                             _P],
    "spand_potrf_batched": [_c_int, _P, _P, _P, _P, _c_int, _c_int, _P],
    "spand_trtri_batched": [_c_int, _P, _P, _P, _P],
    "spand_trtri_tiles": [_c_int, _P, _P, _P, _P],
    "spand_copy_batched": [_c_int, _P, _P, _P, _P],
    "spand_gemm_grouped": [_c_int, _P, _P, _P, _P, _P, _c_dbl, _c_dbl, _c_int,
                           _c_int, _c_int, _P, _c_int, _P],
    "spand_gemm_grouped_masked": [_c_int, _P, _P, _P, _P, _P, _c_dbl, _c_dbl, _c_int,
                                  _c_int, _c_int, _P, _c_int, _P, _P, _P],
    "spand_gemm_kmask": [_c_int, _P, _P, _P, _P, _P, _P, _c_int, _P],
    "spand_rrqr_wave": [_c_int, _c_int, _c_int, _P, _P, _P, _P, _c_dbl, _c_int, _P, _P],
    "spand_rrqr_cta_count": [],
    "spand_rrqr_capacity": [_c_int],
    "spand_rrqr_wave_clustered": [_c_int, _c_int, _c_int, _c_int, _P, _P, _P, _P, _c_dbl,
                                  _c_int, _P, _P],
    "spand_rrqr_cluster_capacity": [_c_int, _c_int],
    "spand_rrqr_max_rows_clustered": [_c_int],
    "spand_plan_set_cluster": [_P, _c_int, _c_int],
    "spand_assemble_final": [_c_int, _P, _c_i64, _P, _P, _P, _c_int, _P, _P],
    "spand_count_nonzero": [_c_int, _P, _P, _P],
    "spand_count_nonzero_pieces": [_c_int, _P, _P, _c_i64, _P, _P, _P, _P],
    "spand_digest_pieces": [_c_int, _P, _P, _P, _P],
    "spand_fv_counts": [_c_int, _P, _P, _P],
    "spand_fv_fill": [_c_int, _P, _c_int, _P, _P, _P, _P, _P],
    "spand_jacobi_prescale": [_c_i64, _P, _P, _P, _P, _P, _P, _P, _P],
    "spand_nd_partition": [_c_i64, _P, _P, _c_int, _P, _P, _P, _P],
    "spand_plan_sizes": [_P, _P],
    "spand_plan_emit": [_P, _c_i64, _c_i64, _c_i64, _c_i64, _c_int],
    "spand_plan_program": [_P, _P, _P],
    "spand_plan_meta": [_P, _P],
    "spand_plan_set_nk": [_P, _c_int],
    "spand_nk_rescale": [_c_int, _P, _P, _P, _P, _c_i64, _c_int, _c_int, _P],
    "spand_nk_basis": [_c_int, _P, _P, _P, _P, _P, _c_i64, _c_int, _c_dbl, _P],
    "spand_nk_deflate": [_c_int, _c_i64, _P, _P, _P, _P, _c_int, _P],
    "spand_nk_qform": [_c_int, _c_i64, _P, _P, _c_int, _P],
}

_lib = None


def load(path=LIB_PATH):
    """Load (once) and type the shared library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is not built; run `python -m "
            f"paper_2007_00789_b200.build_native` (nvcc, sm_100a)")
    lib = ctypes.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = _c_int
    _lib = lib
    return lib


# launches issued through call(), per entry point (bench.py's gpu_launches)
COUNTS = {}
# optional per-entry-point CUDA-event timing (profile() context manager)
_PROFILE = None
_PROFILE_NAMES = None

# host-only entry points (no kernel launch)
_HOST_ONLY = {"spand_plan_sizes", "spand_plan_emit", "spand_plan_program",
              "spand_plan_meta", "spand_nd_partition", "spand_version", "spand_device_sm_count",
              "spand_rrqr_cta_count", "spand_rrqr_capacity", "spand_spmv_blocks", "spand_dot_blocks"}

# entry points issuing several kernels whose callers count them per kernel
_COUNTED_BY_CALLER = {"spand_apply_pass", "spand_run_launches", "spand_apply_pass_persistent"}
_HOST_ONLY |= {"spand_launch_timer_reset", "spand_launch_timer_read"}


def call(name, *args):
    """Invoke an entry point; nonzero status raises RuntimeError."""
    fn = getattr(load(), name)
    if (_PROFILE is not None and name not in _HOST_ONLY
            and (_PROFILE_NAMES is None or name in _PROFILE_NAMES) and not _capturing()):
        import torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = fn(*args)
        e1.record()
        _PROFILE.append((name, e0, e1))
    else:
        st = fn(*args)
    if st != 0:
        raise RuntimeError(f"{name} failed with status {st}")
    if name not in _HOST_ONLY and name not in _COUNTED_BY_CALLER:
        COUNTS[name] = COUNTS.get(name, 0) + 1
    return st


def _capturing():
    import torch
    return torch.cuda.is_current_stream_capturing()


def launches():
    return sum(COUNTS.values())


def profile_mask(type_names):
    """Launch-type bit mask of the native launcher for the active profile()
    (0: none): every type, or those whose entry point is profiled."""
    if _PROFILE is None or _capturing():
        return 0
    mask = 0
    for typ, nm in type_names.items():
        if _PROFILE_NAMES is None or nm in _PROFILE_NAMES:
            mask |= 1 << typ
    return mask


class profile:
    """Context manager: per-entry-point device time (ms) on the current
    stream, measured with CUDA events around every call() (or only around
    the entry points in ``names``: events around ~10k launches per step cost
    host time and launch gaps, so a timed region profiles only the kernel
    whose roofline it reports)."""

    def __init__(self, names=None):
        self.names = None if names is None else set(names)

    def __enter__(self):
        global _PROFILE, _PROFILE_NAMES
        _PROFILE = []
        _PROFILE_NAMES = self.names
        self.result = {}
        load().spand_launch_timer_reset()
        return self

    def __exit__(self, *exc):
        global _PROFILE
        import torch
        torch.cuda.synchronize()
        out = {}
        for name, e0, e1 in _PROFILE:
            if name == "spand_run_launches":
                continue
            ms = e0.elapsed_time(e1)
            tot, cnt = out.get(name, (0.0, 0))
            out[name] = (tot + ms, cnt + 1)
        # launches issued by the native program launcher (timed there)
        import numpy as np
        from .engine import LAUNCH_NAMES
        ms = np.zeros(32)
        n = np.zeros(32, dtype=np.int64)
        load().spand_launch_timer_read(ms.ctypes.data, n.ctypes.data)
        for typ, nm in LAUNCH_NAMES.items():
            if n[typ]:
                tot, cnt = out.get(nm, (0.0, 0))
                out[nm] = (tot + float(ms[typ]), cnt + int(n[typ]))
        _PROFILE = None
        self.result = {k: {"ms": round(v[0], 3), "calls": v[1]} for k, v in
                       sorted(out.items(), key=lambda kv: -kv[1][0])}
        return False
