timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_base2.log 2>&1; echo base_rc=$?
head -6 gpurun_out/waves_base2.log
SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_minb1.so timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_minb1.log 2>&1; echo minb1_rc=$?
head -6 gpurun_out/waves_minb1.log
