"""ctypes binding of the C-ABI in include/spand_b200.h.

The library is REQUIRED: importing a numerical entry point without it (or
without a CUDA device) raises NativeUnavailable; there is no host fallback.
"""

import ctypes
import os

from .errors import NativeUnavailable

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspand_b200.so")

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
    "spand_apply_scatter": [_c_int, _P, _P, _P, _P, _P, _c_i64, _P, _c_i64,
                            _c_int, _P],
    "spand_potrf_batched": [_c_int, _P, _P, _P, _P, _P],
    "spand_trtri_batched": [_c_int, _P, _P, _P, _P],
    "spand_copy_batched": [_c_int, _P, _P, _P, _P],
    "spand_gemm_grouped": [_c_int, _P, _P, _P, _P, _P, _c_dbl, _c_dbl, _c_int,
                           _c_int, _P],
    "spand_rrqr_wave": [_c_int, _c_int, _c_int, _P, _P, _P, _P, _c_dbl, _c_int, _P, _P],
    "spand_rrqr_cta_count": [],
    "spand_assemble_final": [_c_int, _P, _c_i64, _P, _P, _P, _c_int, _P, _P],
    "spand_count_nonzero": [_c_int, _P, _P, _P],
    "spand_nd_partition": [_c_i64, _P, _P, _c_int, _P, _P, _P, _P],
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


def call(name, *args):
    """Invoke an entry point; nonzero status raises RuntimeError."""
    st = getattr(load(), name)(*args)
    if st != 0:
        raise RuntimeError(f"{name} failed with status {st}")
    return st
