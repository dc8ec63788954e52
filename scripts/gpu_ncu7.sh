python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_trunc_warp --csv --log-file gpurun_out/tw_launches.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu7a.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/tw_launches.csv')) if len(r)>5]
h=rows[0]; vi=h.index('Metric Value'); ui=h.index('Metric Unit')
def t(r):
    v=float(r[vi].replace(',','')); return v*1e3 if r[ui]=='usecond' else v*1e6 if r[ui]=='msecond' else v
ts=[t(r) for r in rows[1:]]
i=max(range(len(ts)), key=lambda k: ts[k])
open('gpurun_out/tw_big_index.txt','w').write(str(i))
print(i, ts[i])
PY
IDX=$(cat gpurun_out/tw_big_index.txt)
ncu --set full --clock-control none --import-source on -k regex:k_trunc_warp -s $IDX -c 1 -o gpurun_out/prof_twarp2 python scripts/factor_once.py cfg5 > gpurun_out/ncu7b.log 2>&1
echo done
