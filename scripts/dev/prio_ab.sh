set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -n 3 gpurun_out/tgpu.log
for i in 1 2; do
ACR_NO_PRIO=1 ACR_BENCH_PRIO=0 python bench.py --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noprio', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['passes_ms_per_step'], d['e2e']['solve_ms'])"
python bench.py --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prio', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['passes_ms_per_step'], d['e2e']['solve_ms'])"
done
ACR_FWD_LAG=3 python bench.py --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prio lag3', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['passes_ms_per_step'], d['e2e']['solve_ms'])"
ACR_FWD_LAG=1 python bench.py --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prio lag1', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['passes_ms_per_step'], d['e2e']['solve_ms'])"
