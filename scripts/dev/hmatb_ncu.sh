set -x
ACR_HMATB_SM=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_hmatB --csv --log-file gpurun_out/hb_old.csv python scripts/factor_once.py cfg5 1 > gpurun_out/hb_old.log 2>&1
ACR_HMAT_MINB=5 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_hmatB --csv --log-file gpurun_out/hb_new.csv python scripts/factor_once.py cfg5 1 > gpurun_out/hb_new.log 2>&1
