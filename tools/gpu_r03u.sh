timeout 900 python -m pytest tests/test_gpu_gemm_shapes.py -q -m gpu -x > gpurun_out/pytest_gpu_r03u.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_gpu_r03u.log | grep -v "^frame"
