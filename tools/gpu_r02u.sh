timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_factorize.py tests/test_gpu_multirhs.py tests/test_gpu_contract.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/t_u.log 2>&1; echo rc=$?; tail -2 gpurun_out/t_u.log; grep -E "^FAILED|Error" gpurun_out/t_u.log | head -5
timeout 300 python tools/apply_time.py C4 15 2>&1 | tail -2 | cut -c1-300
true
