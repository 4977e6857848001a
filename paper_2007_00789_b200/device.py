"""Device plumbing: CUDA availability, streams, device CSR, vector moves.

PyTorch owns all device memory (tensors); the C-ABI only sees raw pointers
and the current stream's handle.  Every numerical entry point goes through
``require_cuda()`` so a box without a B200 (or without the built extension)
fails loudly instead of computing on the host.
"""

import ctypes

import numpy as np

from . import _lib
from .errors import DimensionMismatch, NativeUnavailable

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    """Load the extension and make sure a CUDA device is present."""
    _lib.load()
    t = torch()
    if not t.cuda.is_available():
        raise NativeUnavailable(
            "no CUDA device: the spaND kernels run only on the GPU "
            "(no host fallback)")
    return t


def dev():
    return torch().device("cuda", torch().cuda.current_device())


def stream():
    """Raw cudaStream_t of torch's current stream (as a c_void_p)."""
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def to_dev(arr, dtype=None):
    """numpy -> device tensor (contiguous)."""
    t = torch()
    a = np.ascontiguousarray(arr if dtype is None else arr.astype(dtype))
    return t.from_numpy(a).to(dev(), non_blocking=False)


class PinnedArena:
    """Grow-only pinned host staging for asynchronous uploads.  Regions are
    handed out sequentially and recycled by ``reset()``, which callers issue
    only after a device synchronisation (so no copy still reads them)."""

    def __init__(self):
        self.buf = None
        self.at = 0

    def reset(self):
        self.at = 0

    def take(self, nbytes):
        t = torch()
        need = self.at + nbytes
        if self.buf is None or need > self.buf.numel():
            # a new (larger) block: earlier regions keep their old buffer
            # alive through the tensors that reference them
            size = max(need, 2 * (self.buf.numel() if self.buf is not None else 0), 1 << 24)
            self.buf = t.empty(size, dtype=t.uint8, pin_memory=True)
            self.at = 0
            need = nbytes
        view = self.buf[self.at:need]
        self.at = (need + 255) // 256 * 256
        return view


ARENA = PinnedArena()


def to_dev_async(arr, dtype=None):
    """numpy -> device tensor without blocking the host: the array is staged
    in the pinned arena and copied with non_blocking=True on the current
    stream, so host-side planning overlaps device work."""
    t = torch()
    a = np.ascontiguousarray(arr if dtype is None else arr.astype(dtype))
    if a.nbytes == 0:
        return t.from_numpy(a).to(dev())
    stage = ARENA.take(a.nbytes)
    host = stage.view(t.from_numpy(a).dtype).view(a.shape)
    host.copy_(t.from_numpy(a))
    out = t.empty(a.shape, dtype=host.dtype, device=dev())
    out.copy_(host, non_blocking=True)
    out._spand_stage = stage   # the staging region outlives the copy
    return out


def as_device_vector(x, n):
    """Accept numpy or torch input of shape (n,) or (n, k); return a
    contiguous fp64 device tensor and a tag telling how to hand back."""
    t = require_cuda()
    if isinstance(x, t.Tensor):
        kind = ("torch", x.device, x.dtype)
        xd = x.to(device=dev(), dtype=t.float64)
    else:
        kind = ("numpy",)
        xd = t.from_numpy(np.array(x, dtype=np.float64, copy=True)).to(dev())
    if xd.shape[0] != n:
        raise DimensionMismatch(
            f"vector has {xd.shape[0]} entries, expected {n}")
    return xd.contiguous(), kind


def like_input(y, kind):
    if kind[0] == "numpy":
        return y.cpu().numpy()
    return y.to(device=kind[1], dtype=kind[2])


class DeviceCSR:
    """CSR on the device: int32 row_ptr/col_idx, fp64 values."""

    def __init__(self, n, row_ptr, col_idx, values):
        self.n = int(n)
        self.nnz = int(values.shape[0])
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values
        t = torch()
        self._pdot = t.empty(max(1, _lib.load().spand_spmv_blocks(self.n)),
                             dtype=t.float64, device=dev())

    @classmethod
    def from_host(cls, a, perm=None):
        """Upload; with ``perm`` (new -> old) build P A P^T in the new order."""
        require_cuda()
        n = a.n
        rp, ci, va = a.row_ptr, a.col_idx, a.values
        if perm is not None:
            perm = np.asarray(perm, dtype=np.int64)
            inv = np.empty(n, dtype=np.int64)
            inv[perm] = np.arange(n)
            counts = np.diff(rp)[perm]
            new_rp = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(counts, out=new_rp[1:])
            src = (np.repeat(rp[perm] - new_rp[:-1], counts)
                   + np.arange(int(new_rp[-1])))
            rows = np.repeat(np.arange(n), counts)
            cols = inv[ci[src]]
            vals = va[src]
            order = np.lexsort((cols, rows))
            rp, ci, va = new_rp, cols[order], vals[order]
        if rp[-1] >= 2 ** 31:
            raise DimensionMismatch("nnz(A) must fit int32 on the device")
        return cls(n, to_dev(rp, np.int32), to_dev(ci, np.int32),
                   to_dev(va, np.float64))

    def spmv(self, x, out=None, pdot=None):
        """y = A x for a device vector (n,) or stack (n, k)."""
        t = torch()
        if out is None:
            out = t.empty_like(x)
        if x.dim() == 1:
            _lib.call("spand_csr_spmv", self.n, ptr(self.row_ptr),
                      ptr(self.col_idx), ptr(self.values), ptr(x), ptr(out),
                      ptr(pdot) if pdot is not None else None, stream())
        else:
            xs = x.t().contiguous()
            ys = t.empty_like(xs)
            for j in range(xs.shape[0]):
                _lib.call("spand_csr_spmv", self.n, ptr(self.row_ptr),
                          ptr(self.col_idx), ptr(self.values), ptr(xs[j]),
                          ptr(ys[j]), None, stream())
            out.copy_(ys.t())
        return out


class nvtx:
    """NVTX range around a host phase (ncu --nvtx / Nsight filters): the
    factorization's symbolic analysis, device program and collection, the
    PCG solve and the apply image build."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        try:
            torch().cuda.nvtx.range_push(self.name)
            self.ok = True
        except Exception:
            self.ok = False
        return self

    def __exit__(self, *exc):
        if self.ok:
            torch().cuda.nvtx.range_pop()
        return False
