for cap in 1 2 8 64; do
  echo "cap=$cap" >> gpurun_out/cap.log
  SPAND_RRQR_CAP=$cap timeout 60 python tools/gpu_factor_one.py lap2d_d16_L4_e0.05_k1_second-full >> gpurun_out/cap.log 2>&1
  SPAND_RRQR_CAP=$cap timeout 60 python tools/gpu_factor_one.py C1_first >> gpurun_out/cap.log 2>&1
done
