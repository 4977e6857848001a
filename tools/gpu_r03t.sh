bash tools/variant_waves.sh mt2 mt4
for v in mt2 mt4; do sed -n 2,4p gpurun_out/waves_$v.log | cut -c1-90; done
SPAND_LIB_PATH=$PWD/paper_2007_00789_b200/variants/libspand_mt4.so timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_factorize.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/pytest_gpu_mt4.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_mt4.log
