timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tall.log 2>&1
echo "exit $?" >> gpurun_out/tall.log
timeout 900 python scripts/time_configs.py cfg1 cfg2 cfg3 cfg5 > gpurun_out/time.log 2>&1
