timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r02l.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_r02l.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r02l.json 2> gpurun_out/bench_r02l.err; echo bench_rc=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_r02l.json').read().strip().splitlines()[-1])
for k in ['value','ms_per_step','factorize_s','solve_s','n_cg','apply','e2e','gpu_launches']: print(k, d.get(k))
print(d['kernels_ms_per_step'])
P
