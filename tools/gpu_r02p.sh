python tools/one_factor.py C4 15 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rrqr_wave_kernel -s 0 -c 1 -o gpurun_out/rrqr_classic_root python tools/one_factor.py C4 15 > gpurun_out/ncu_rc.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_rc.log
