for cfg in "1.5 0.5" "1.0 0.5" "1.25 0.75" "1.25 0.25"; do
set -- $cfg
SPAND_GROUP_WEIGHT=3 SPAND_GROUP_EM=$1 SPAND_GROUP_EN=$2 timeout 300 python tools/waves_twice.py C4 15 > gpurun_out/w_gw.log 2>&1; echo "em=$1 en=$2"; grep -v barrier gpurun_out/w_gw.log | tail -1 | cut -c1-100
done
