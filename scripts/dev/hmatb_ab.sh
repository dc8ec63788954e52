set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -n 12 gpurun_out/tgpu.log
for i in 1 2; do
  ACR_NO_QSPLIT=1 python scripts/factor_once.py cfg5 6 | tail -1
  python scripts/factor_once.py cfg5 6 | tail -1
done
ACR_DEBUG=1 python scripts/factor_once.py cfg5 3 2>&1 | grep host_ms | tail -n 11 | awk '{print $3,$NF}' | tr '\n' ' '
