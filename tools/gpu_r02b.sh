timeout 300 python tools/rrqr_phase_run.py 15 > gpurun_out/phases_r02c.log 2>&1; echo phases_rc=$?
grep "rrqr phases" gpurun_out/phases_r02c.log | awk '{for(i=1;i<=NF;i++) if($i=="m") m=$(i+1); print m, $0}' | sort -n -r | head -6 | cut -c1-420
