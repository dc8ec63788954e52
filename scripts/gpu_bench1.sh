python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "exit $?" >> gpurun_out/bench1.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench1_ref.json 2>> gpurun_out/bench1.err
python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1_cfg2.json 2>> gpurun_out/bench1.err
