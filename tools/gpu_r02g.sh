for v in rho30 rho10 rho03; do
SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_$v.so timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_$v.log 2>&1; echo $v rc=$?
head -4 gpurun_out/waves_$v.log | cut -c1-60
done
