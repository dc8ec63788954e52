# quick iteration: GPU parity tests, then instrumented cfg5 timing
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/tall.log 2>&1; echo "exit $?" >> gpurun_out/tall.log
PROF=1 REPS=3 timeout 600 python scripts/time_configs.py cfg5 > gpurun_out/prof5.log 2>&1
echo "exit $?" >> gpurun_out/prof5.log
