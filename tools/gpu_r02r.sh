SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_lastarr.so timeout 300 python tools/one_factor.py C4 15 > gpurun_out/lastarr.log 2>&1; echo rc=$?
grep "\[last\]" gpurun_out/lastarr.log | sort -t' ' -k10 -n -r | head -40
