set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrqr_wave_kernel -s 0 -c 1 -f -o gpurun_out/rrqr_root_r03 python tools/one_factor.py C4 15 > gpurun_out/ncu_root.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_grouped_kernel -s 222 -c 1 -f -o gpurun_out/gemm_top1_r03 python tools/one_factor.py C4 15 > gpurun_out/ncu_gemm1.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_grouped_kernel -s 386 -c 1 -f -o gpurun_out/gemm_top2_r03 python tools/one_factor.py C4 15 > gpurun_out/ncu_gemm2.log 2>&1; echo rc=$?
ls -la gpurun_out/*.ncu-rep
