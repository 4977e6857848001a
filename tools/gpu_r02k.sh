SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_dfstats.so timeout 300 python tools/apply_time.py C4 15 > gpurun_out/dfstats.log 2>&1; echo rc=$?
grep -v "^\[df\]" gpurun_out/dfstats.log | tail -3 | cut -c1-300
grep "^\[df\]" gpurun_out/dfstats.log | head -4736 > gpurun_out/dfstats_one.log
python tools/df_stats.py gpurun_out/dfstats_one.log
