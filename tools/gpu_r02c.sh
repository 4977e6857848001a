set -x
timeout 600 python -m pytest tests/test_gpu_rrqr_cluster.py -x -q -m gpu > gpurun_out/cl_tests.log 2>&1; echo rc=$?
tail -30 gpurun_out/cl_tests.log
timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_cl.log 2>&1; echo waves_rc=$?
head -25 gpurun_out/waves_cl.log
