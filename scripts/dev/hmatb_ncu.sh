set -x
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gp_tc|k_hmatA_tc<" --csv --log-file gpurun_out/ga_new.csv python scripts/factor_once.py cfg5 1 > gpurun_out/ga_new.log 2>&1
