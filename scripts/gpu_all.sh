timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/tall.log 2>&1
echo "exit $?" >> gpurun_out/tall.log
