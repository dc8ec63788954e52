# full round check: tests, smoke, bench (both arms), launch list
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/tall.log 2>&1; echo "exit $?" >> gpurun_out/tall.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
