timeout 1500 python -m pytest tests/test_gpu_gemm_shapes.py tests/test_gpu_kernels.py tests/test_gpu_factorize.py tests/test_gpu_configs.py tests/test_gpu_contract.py -q -m gpu -x > gpurun_out/pytest_gpu_r03p.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r03p.log
timeout 900 python bench.py --no-cpu-baseline --no-near-kernel --steps 3 --warmup 3 > gpurun_out/bench_r03p.json 2> gpurun_out/bench_r03p.err; echo bench_rc=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_r03p.json').read().strip().splitlines()[-1])
for k in ['value','ms_per_step','factorize_s','solve_s','n_cg']: print(k, d.get(k))
print(d['kernels_ms_per_step'])
P
