timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tall.log 2>&1
echo "exit $?" >> gpurun_out/tall.log
for v in 0 1 2 3; do
  echo "variant $v" >> gpurun_out/ab.log
  ACR_PAIR=$v PROF=1 REPS=3 python scripts/time_configs.py cfg5 2>&1 | cut -c1-2000 >> gpurun_out/ab.log
done
