PROF=1 REPS=3 python scripts/time_configs.py cfg2 cfg5 > gpurun_out/prof.log 2>&1
