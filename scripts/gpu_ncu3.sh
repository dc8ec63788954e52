python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_cfg5_v6.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu_cfg5.log 2>&1
echo done
