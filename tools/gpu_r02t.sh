timeout 900 python -m pytest tests/test_gpu_apply.py tests/test_gpu_factorize.py tests/test_gpu_multirhs.py tests/test_gpu_contract.py -q -m gpu -x > gpurun_out/t_t.log 2>&1; echo rc=$?; tail -2 gpurun_out/t_t.log
timeout 300 python tools/apply_time.py C4 15 2>&1 | tail -2 | cut -c1-400
timeout 300 python tools/step_timeline.py 2>&1 | tail -2 | cut -c1-300
