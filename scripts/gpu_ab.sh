timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tall.log 2>&1
echo "exit $?" >> gpurun_out/tall.log
REPS=4 python scripts/time_configs.py cfg2 cfg5 2>&1 | cut -c1-2000 >> gpurun_out/ab.log
