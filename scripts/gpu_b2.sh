python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/b2_cfg5.json 2> gpurun_out/b2.err
python bench.py --config cfg2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b2_cfg2.json 2>> gpurun_out/b2.err
