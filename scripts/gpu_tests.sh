# GPU tests (run under gpurun); extra pytest arguments are passed through
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -q -m gpu -x "$@" > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -30 gpurun_out/tgpu.log
