timeout 300 python tools/waves_twice.py C4 15 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_contract.py -q -m gpu -x > gpurun_out/cfg_q.log 2>&1; echo rc=$?; tail -2 gpurun_out/cfg_q.log
