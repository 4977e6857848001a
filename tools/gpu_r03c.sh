timeout 600 python tools/step_timeline.py > gpurun_out/timeline_r03c.log 2>&1; echo rc=$?
tail -3 gpurun_out/timeline_r03c.log
timeout 1500 python -m pytest tests/test_gpu_rrqr_cluster.py tests/test_gpu_schemes.py tests/test_near_kernel.py tests/test_elasticity.py tests/test_local_errors.py -q -m gpu > gpurun_out/pytest_gpu_r03c.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r03c.log
