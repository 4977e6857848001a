for i in 1 2 3 4 5 6; do
SPAND_RRQR_DEBUG=1 timeout 60 python tools/gpu_factor_one.py lap2d_d16_L4_e0.05_k1_first >> gpurun_out/race.log 2>&1
SPAND_RRQR_DEBUG=1 timeout 60 python tools/gpu_factor_one.py lap2d_d16_L4_e0.05_k1_second-full >> gpurun_out/race.log 2>&1
done
