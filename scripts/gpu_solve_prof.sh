python scripts/solve_once.py > gpurun_out/solve_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py > gpurun_out/solve_ncu.log 2>&1
echo done
