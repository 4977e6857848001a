timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r02x.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r02x.log
