export SPAND_RRQR_CLUSTER=8
python tools/one_factor.py C4 15 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:rrqr_wave_kernel --csv --log-file gpurun_out/rrqr_cl_list.csv python tools/one_factor.py C4 15 > gpurun_out/ncu_list.log 2>&1; echo list_rc=$?
IDX=$(python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/rrqr_cl_list.csv')) if len(r)>10]
hdr=rows[0]; ii=hdr.index('ID'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value')
d={}
for r in rows[1:]:
    if r[mi]=='gpu__time_duration.sum': d[int(r[ii])]=float(r[vi].replace(',',''))
ids=sorted(d); best=max(d,key=d.get); print(ids.index(best))
P
)
echo root_index=$IDX
ncu --set full --clock-control none --import-source on -k regex:rrqr_wave_kernel -s $IDX -c 1 -o gpurun_out/rrqr_cl_root python tools/one_factor.py C4 15 > gpurun_out/ncu_cl.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu_cl.log
