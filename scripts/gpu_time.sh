timeout 1500 python scripts/time_configs.py cfg1 cfg2 cfg3 cfg4 cfg5 > gpurun_out/time.log 2>&1
echo "exit $?" >> gpurun_out/time.log
