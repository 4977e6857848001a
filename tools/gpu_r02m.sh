timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r02m.json 2> gpurun_out/bench_r02m.err; echo bench_rc=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_r02m.json').read().strip().splitlines()[-1])
for k in ['value','ms_per_step','factorize_s','solve_s','n_cg','apply','e2e','gpu_launches','nnz_factor']: print(k, d.get(k))
print(d['kernels_ms_per_step'])
P
timeout 300 python tools/step_timeline.py > gpurun_out/timeline_r02m.log 2>&1; tail -30 gpurun_out/timeline_r02m.log
