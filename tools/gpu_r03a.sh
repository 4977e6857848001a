timeout 300 python tools/q_zero_pattern.py hc3d_d16_L8_e0.01_k2_second-full lap2d_d32_L5_e0.01_k1_second-full hc2d_d64_L8_e0.01_k4_second-full > gpurun_out/qzero.log 2>&1; echo qzero_rc=$?
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_r03a.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_r03a.log
timeout 900 python bench.py > gpurun_out/bench_r03a.json 2> gpurun_out/bench_r03a.err; echo bench_rc=$?
tail -c 600 gpurun_out/bench_r03a.err
