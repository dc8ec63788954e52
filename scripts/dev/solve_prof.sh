# launch list of one 16-RHS solve (after a plain factor) and of a fused factor+backsub
set -x
python scripts/factor_once.py cfg5 6 | tail -1
ACR_LEAFINV_4=0 python scripts/factor_once.py cfg5 6 | tail -1
python scripts/factor_once.py cfg5 6 | tail -1
ACR_LEAFINV_4=0 python scripts/factor_once.py cfg5 6 | tail -1
python scripts/solve_once.py cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py cfg5 > gpurun_out/solve_ncu.log 2>&1
python scripts/gap_probe.py cfg5 > gpurun_out/gap_probe.txt 2>&1
tail -n 40 gpurun_out/gap_probe.txt
