timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_r02s.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r02s.log
timeout 900 python bench.py > gpurun_out/bench_r02s.json 2> gpurun_out/bench_r02s.err; echo bench_rc=$?
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 12000 --csv --log-file gpurun_out/launches_r02s.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
