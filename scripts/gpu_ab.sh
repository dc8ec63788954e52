timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tall.log 2>&1
echo "exit $?" >> gpurun_out/tall.log
PROF=1 REPS=3 python scripts/time_configs.py cfg5 2>&1 | cut -c1-2000 >> gpurun_out/ab.log
python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_leafinv" --csv --log-file gpurun_out/sm_launches.csv python scripts/factor_once.py cfg5 > /dev/null 2>&1
