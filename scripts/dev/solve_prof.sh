set -x
python scripts/solve_once.py cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py cfg5 > gpurun_out/solve_ncu.log 2>&1
