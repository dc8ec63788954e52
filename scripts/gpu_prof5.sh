PROF=1 REPS=2 timeout 600 python scripts/time_configs.py cfg5 > gpurun_out/prof5.log 2>&1
echo "exit $?" >> gpurun_out/prof5.log
