#!/bin/bash
# build_variant.sh NAME "NVCC DEFINES" : rrqr.cu with extra defines, linked with the
# regular objects into paper_2007_00789_b200/variants/libspand_NAME.so
set -e
cd "$(dirname "$0")/../paper_2007_00789_b200/csrc"
mkdir -p ../variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $2 -c rrqr.cu -o /tmp/rrqr_$1.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/libspand_$1.so $(ls build/*.o | grep -v rrqr.cu.o) /tmp/rrqr_$1.o -lcudart
echo built ../variants/libspand_$1.so
