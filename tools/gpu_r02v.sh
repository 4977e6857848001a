timeout 900 python bench.py > gpurun_out/bench_r02v.json 2> gpurun_out/bench_r02v.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02v.json 2> gpurun_out/bench_ref_r02v.err; echo ref_rc=$?
