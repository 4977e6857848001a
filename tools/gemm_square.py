"""Square-GEMM throughput of the grouped DMMA kernel (spand_gemm_grouped)
against cuBLAS DGEMM on the same device, C = A B^T (the Schur-update form)."""
import json, sys
sys.path.insert(0, '.')
import torch
from paper_2007_00789_b200.kernels import Geometry, gemm_grouped, opnd
for n in (1024, 2048, 4096):
    geo = Geometry.virtual([n, n, n])
    a = torch.randn(n * n, dtype=torch.float64, device="cuda")
    b = torch.randn(n * n, dtype=torch.float64, device="cuda")
    c = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    tgt = [(opnd(c.data_ptr(), 0, 2), [(opnd(a.data_ptr(), 0, 1), opnd(b.data_ptr(), 2, 1))], (n, n))]
    gemm_grouped(geo, tgt, 1.0, 0.0, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        gemm_grouped(geo, tgt, 1.0, 0.0, 1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    A = a.view(n, n); B = b.view(n, n)
    C = A @ B.T
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        C = A @ B.T
    e1.record(); torch.cuda.synchronize()
    ms_cb = e0.elapsed_time(e1) / reps
    ref = (A.T @ B).T   # column-major view: c[i + j n] = sum_k a[i + k n] b[j + k n]
    got = c.view(n, n)
    err = (got - (B.T.T @ A.T.T).T).abs().max().item() if n <= 1024 else None
    print(json.dumps({"n": n, "spand_ms": ms, "spand_tflops": 2 * n ** 3 / ms / 1e9,
                      "cublas_ms": ms_cb, "cublas_tflops": 2 * n ** 3 / ms_cb / 1e9}))
