timeout 600 python tools/prof_waves.py C4 15 > gpurun_out/waves_r03h.log 2>&1; echo rc=$?
head -3 gpurun_out/waves_r03h.log
timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_factorize.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/pytest_gpu_r03h.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r03h.log
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 12000 --csv --log-file gpurun_out/launches_r03h.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
