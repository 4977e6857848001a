for v in gm1 gm4 gm5; do
  SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_$v.so timeout 600 python bench.py --no-cpu-baseline --no-near-kernel --steps 3 --warmup 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
  python - <<P
import json
d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],1), d['kernels_ms_per_step']['spand_gemm_grouped'], d['kernels_ms_per_step']['spand_rrqr_wave'], d['n_cg'])
P
done
timeout 600 python tools/nnz_small.py --all > gpurun_out/nnz_small.log 2>&1; tail -30 gpurun_out/nnz_small.log
