timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_factorize.py tests/test_gpu_multirhs.py -x -q -m gpu > gpurun_out/apply_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/apply_tests.log
timeout 300 python tools/apply_time.py C4 15 2>&1 | tail -2
SPAND_APPLY_DATAFLOW=0 timeout 300 python tools/apply_time.py C4 15 2>&1 | tail -2
