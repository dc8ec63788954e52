ACR_DEBUG=1 REPS=3 python scripts/time_configs.py cfg5 > gpurun_out/dbg.log 2>&1
