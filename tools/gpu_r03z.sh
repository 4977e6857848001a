timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_r03z.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r03z.log
timeout 900 python bench.py > gpurun_out/bench_r03z.json 2> gpurun_out/bench_r03z.err; echo bench_rc=$?
tail -c 300 gpurun_out/bench_r03z.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r03z.json 2> gpurun_out/bench_ref_r03z.err; echo ref_rc=$?
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 16000 --csv --log-file gpurun_out/launches_r03z.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
