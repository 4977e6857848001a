timeout 900 python -m pytest tests/test_gpu_gemm_shapes.py tests/test_gpu_factorize.py -q -m gpu -x > gpurun_out/pytest_gpu_r03i.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_gpu_r03i.log
timeout 900 python bench.py --no-cpu-baseline --no-near-kernel --steps 3 --warmup 3 > gpurun_out/bench_r03i.json 2> gpurun_out/bench_r03i.err; echo bench_rc=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_r03i.json').read().strip().splitlines()[-1])
for k in ['value','ms_per_step','factorize_s','solve_s','n_cg']: print(k, d.get(k))
print(d['kernels_ms_per_step'])
P
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:rrqr_wave_kernel --csv --log-file gpurun_out/rrqr_dram_r03.csv python tools/one_factor.py C4 15 > gpurun_out/ncu_dram.log 2>&1; echo ncu_rc=$?
