import os
import sys

# the oracle is pinned bitwise to fixtures frozen with one BLAS thread
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


try:  # numpy may already be loaded by a plugin: pin OpenBLAS at runtime too
    from threadpoolctl import threadpool_limits
    _BLAS_LIMIT = threadpool_limits(limits=1, user_api="blas")
except Exception:  # pragma: no cover
    _BLAS_LIMIT = None
