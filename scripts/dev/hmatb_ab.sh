set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -n 3 gpurun_out/tgpu.log
for i in 1 2; do
  ACR_HMATB_SM=1 python scripts/factor_once.py cfg5 6 | tail -1
  python scripts/factor_once.py cfg5 6 | tail -1
done
python scripts/solve_once.py cfg5
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_hmatB --csv --log-file gpurun_out/hb_new.csv python scripts/factor_once.py cfg5 1 > gpurun_out/hb_new.log 2>&1
for lag in 3 4 6 7; do ACR_FWD_LAG=$lag python bench.py --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag $lag', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['solve_ms'])"; done
python bench.py --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag default', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['solve_ms'])"
