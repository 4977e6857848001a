set -x
timeout 600 python tools/scheme_diff.py 64 0.01 first second-superfine > gpurun_out/scheme_diff.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_factorize.py -q -m gpu -rf -x > gpurun_out/pytest_contract.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests/test_gpu_configs.py -q -m gpu -rf -s -k c3_every > gpurun_out/pytest_c3.log 2>&1; echo rc=$?
