set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -n 3 gpurun_out/tgpu.log
for i in 1 2 3; do
  python scripts/factor_once.py cfg5 6 | tail -1
done
python scripts/solve_once.py cfg5
