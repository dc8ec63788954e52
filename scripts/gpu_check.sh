# round check on one B200: GPU tests, smoke, bench (run under gpurun)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/tall.log 2>&1; echo "exit $?" >> gpurun_out/tall.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/tall.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/bench.json | head -c 600
