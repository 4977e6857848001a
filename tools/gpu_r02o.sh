python tools/one_factor.py C4 15 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:gemm_grouped --csv --log-file gpurun_out/gemm_list.csv python tools/one_factor.py C4 15 > gpurun_out/ncu_glist.log 2>&1; echo list_rc=$?
IDX=$(python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/gemm_list.csv')) if len(r)>10]
hdr=rows[0]; ii=hdr.index('ID'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value')
d={}
for r in rows[1:]:
    if r[mi]=='gpu__time_duration.sum': d[int(r[ii])]=float(r[vi].replace(',',''))
ids=sorted(d); top=sorted(d,key=d.get,reverse=True)[:3]
print(' '.join(str(ids.index(t)) for t in top))
P
)
echo top=$IDX
set -- $IDX
ncu --set full --clock-control none --import-source on -k regex:gemm_grouped -s $1 -c 1 -o gpurun_out/gemm_top1 python tools/one_factor.py C4 15 > gpurun_out/ncu_g1.log 2>&1; echo g1=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_grouped -s $2 -c 1 -o gpurun_out/gemm_top2 python tools/one_factor.py C4 15 > gpurun_out/ncu_g2.log 2>&1; echo g2=$?
