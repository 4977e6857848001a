SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_r1rrqr.so timeout 300 python tools/waves_twice.py C4 15 > gpurun_out/w_r1rrqr.log 2>&1; echo r1; tail -1 gpurun_out/w_r1rrqr.log
timeout 300 python tools/waves_twice.py C4 15 2>&1 | tail -1
