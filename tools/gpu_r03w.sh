bash tools/variant_waves.sh base0 rd6 rd9 rc5 rc8 b04 b016 ra5 ra2 base0
