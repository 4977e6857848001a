set -x
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=10 -s -k "contract or configs" > gpurun_out/pytest_contract.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests -q -m gpu -rf --durations=5 -k "not contract and not configs" > gpurun_out/pytest_rest.log 2>&1; echo rc=$?
timeout 600 python tools/payload_diff.py C3 12 > gpurun_out/payload_diff_c3.log 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.log 2>&1; echo rc=$?
