bash tools/variant_waves.sh ru2 ru4
for v in ru2 ru4; do head -3 gpurun_out/waves_$v.log | tail -2; done
