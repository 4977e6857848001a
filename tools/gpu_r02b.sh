timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_r02b.log 2>&1; echo waves_rc=$?
timeout 300 python tools/rrqr_phase_run.py 15 > gpurun_out/phases_r02b.log 2>&1; echo phases_rc=$?
head -30 gpurun_out/waves_r02b.log
grep "rrqr phases" gpurun_out/phases_r02b.log | sort -t' ' -k5 -n -r | head -30
