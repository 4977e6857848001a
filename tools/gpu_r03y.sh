bash tools/variant_waves.sh cw
timeout 300 python tools/prof_waves.py C4 15 > gpurun_out/waves_main.log 2>&1; echo "main $(head -1 gpurun_out/waves_main.log)"
bash tools/variant_waves.sh cw
python - <<'P'
import json
def load(f):
    r=[json.loads(l) for l in open(f).read().strip().splitlines()[1:]]
    return r
a=load('gpurun_out/waves_main.log'); b=load('gpurun_out/waves_cw.log')
ka={(x['npanel'],x['m_max'],x['n_max']):x['ms'] for x in a}
for x in b:
    k=(x['npanel'],x['m_max'],x['n_max'])
    if k in ka and x['npanel']>=10: print(k, ka[k], '->', x['ms'])
P
