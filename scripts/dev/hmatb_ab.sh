set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -n 5 gpurun_out/tgpu.log
for i in 1 2; do
  ACR_HMATB_SM=1 python scripts/factor_once.py cfg5 6 | tail -1
  python scripts/factor_once.py cfg5 6 | tail -1
done
ACR_HMATB_SM=1 ACR_NO_SOLVE_DIAG=1 python scripts/solve_once.py cfg5
ACR_NO_SOLVE_DIAG=1 python scripts/solve_once.py cfg5
python scripts/solve_once.py cfg5
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_hmatB --csv --log-file gpurun_out/hb_new.csv python scripts/factor_once.py cfg5 1 > gpurun_out/hb_new.log 2>&1
python bench.py > gpurun_out/bench_dev.json 2> gpurun_out/bench_dev.err
cat gpurun_out/bench_dev.json
