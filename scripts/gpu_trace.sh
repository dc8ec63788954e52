ACR_TRACE_TRUNC=1 REPS=1 python scripts/time_configs.py cfg5 > gpurun_out/tr.log 2> gpurun_out/tr.err
