bash tools/variant_waves.sh rb1 rb2 rb4
for v in rb1 rb2 rb4; do sed -n 2,3p gpurun_out/waves_$v.log; done
