set -x
timeout 900 python -m pytest tests/test_gpu_rrqr_cluster.py -x -q -m gpu > gpurun_out/cl_tests.log 2>&1; echo rc=$?
grep -v "barrier timeout" gpurun_out/cl_tests.log | tail -15
timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_cl.log 2>&1; echo waves_rc=$?
head -12 gpurun_out/waves_cl.log
