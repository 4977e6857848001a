#!/bin/bash
# tools/variant_waves.sh NAME... : RRQR total of C4-L15 with each variant library
for v in "$@"; do
  SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_$v.so timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_$v.log 2>&1
  echo "$v $(head -1 gpurun_out/waves_$v.log)"
done
