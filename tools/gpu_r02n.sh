for v in blk0_1 blk0_4 blk0_8; do
SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_$v.so timeout 300 python tools/waves_twice.py C4 15 > gpurun_out/w_$v.log 2>&1; echo $v; tail -1 gpurun_out/w_$v.log
done
timeout 300 python tools/waves_twice.py C4 15 2>&1 | tail -1
