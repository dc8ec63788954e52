ACR_DEBUG=1 timeout 300 python -m pytest tests -x -q -s -m gpu -k "kernel_vectors or rand_m4 or rand_m5" > gpurun_out/t2.log 2>&1
echo "exit $?" >> gpurun_out/t2.log
