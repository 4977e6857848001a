"""cuBLAS DGEMM reference point for the FP64 roofline (torch.matmul float64).

Prints one JSON line per size: best-of-10 CUDA-event time, TFLOP/s.
"""
import json
import torch

dev = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b)
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"probe": "cublas_dgemm", "n": n, "ms": best,
                      "tflops": 2 * n ** 3 / best / 1e9}))
