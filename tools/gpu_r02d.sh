timeout 300 python tools/rrqr_phase_run.py 15 > gpurun_out/phases_cl.log 2>&1; echo phases_rc=$?
grep "rrqr phases" gpurun_out/phases_cl.log | awk '{for(i=1;i<=NF;i++) if($i=="m") m=$(i+1); print m, $0}' | sort -n -r | head -6 | cut -c1-420
grep "rrqr cl" gpurun_out/phases_cl.log | awk '{for(i=1;i<=NF;i++) if($i=="m") m=$(i+1); print m, $0}' | sort -n -r | head -12
timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_cl.log 2>&1; echo waves_rc=$?
head -8 gpurun_out/waves_cl.log
