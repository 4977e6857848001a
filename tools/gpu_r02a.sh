set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu_r02a.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/pytest_gpu_r02a.log
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_r02a.json
