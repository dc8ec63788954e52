nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "kernel_vectors or small_systems" > gpurun_out/t1.log 2>&1
echo "exit $?" >> gpurun_out/t1.log
