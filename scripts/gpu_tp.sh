timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tall.log 2>&1
echo "exit $?" >> gpurun_out/tall.log
PROF=1 REPS=4 python scripts/time_configs.py cfg2 cfg5 > gpurun_out/prof.log 2>&1
python scripts/solve_once.py >> gpurun_out/prof.log 2>&1
