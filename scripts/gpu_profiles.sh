# launch list + ncu full captures of the current top kernels (cfg5 factor)
python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_cfg5_v2.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu_l.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_cfg5_v2.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
def t(r):
    v=float(r[vi].replace(',','')); return v*1e3 if r[ui]=='usecond' else v*1e6 if r[ui]=='msecond' else v
idx={}
for name in ['k_trunc_warp','k_trunc_big','k_hmatB_path','k_leafgemm_tc','k_leafinv_reg']:
    ks=[(i,t(r)) for i,r in enumerate(rows[1:]) if name in r[ki]]
    j=max(range(len(ks)), key=lambda q: ks[q][1]) if ks else 0
    idx[name]=j
open('gpurun_out/prof_idx.txt','w').write('\n'.join(f'{k} {v}' for k,v in idx.items()))
PY
while read K I; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s $I -c 1 -o gpurun_out/p2_$K python scripts/factor_once.py cfg5 > gpurun_out/ncu_$K.log 2>&1
done < gpurun_out/prof_idx.txt
echo done
