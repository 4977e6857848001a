python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 14000 --csv --log-file gpurun_out/launches_r03q.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-near-kernel > gpurun_out/ncu_launch.log 2>&1; echo ncu_rc=$?
