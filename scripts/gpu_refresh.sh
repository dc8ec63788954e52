# bench lines (both arms), launch list and ncu --set full captures of the top kernels (cfg5)
V=${V:-v7}
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$V.json 2>> gpurun_out/bench_$V.err
python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_cfg5_$V.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu_l.log 2>&1
python - <<'PY'
import csv, os
V = os.environ.get("V", "v7")
rows=[r for r in csv.reader(open(f'gpurun_out/launches_cfg5_{V}.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
def t(r):
    v=float(r[vi].replace(',','')); return v*1e3 if r[ui]=='usecond' else v*1e6 if r[ui]=='msecond' else v
idx={}
for name in ['k_trunc_warp','k_trunc_big']:
    ks=[(i,t(r)) for i,r in enumerate(rows[1:]) if name in r[ki]]
    j=max(range(len(ks)), key=lambda q: ks[q][1]) if ks else 0
    idx[name]=j
open('gpurun_out/prof_idx.txt','w').write(''.join(f'{k} {v}\n' for k,v in idx.items()))
PY
while read K I; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s $I -c 1 -o gpurun_out/${V}_$K -f python scripts/factor_once.py cfg5 > gpurun_out/ncu_$K.log 2>&1 < /dev/null
done < gpurun_out/prof_idx.txt
echo done > gpurun_out/refresh_done
