timeout 600 python tools/prof_waves.py C4 15 > gpurun_out/waves_r03f.log 2>&1; echo rc=$?
head -4 gpurun_out/waves_r03f.log
timeout 600 python tools/rrqr_phase_run.py 15 > gpurun_out/phases_r03f.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_factorize.py -q -m gpu -x > gpurun_out/pytest_gpu_r03f.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r03f.log
