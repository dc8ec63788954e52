python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_leafinv -s 345 -c 1 -o gpurun_out/prof_linv3 python scripts/factor_once.py cfg5 > gpurun_out/ncu6.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_leafinv --csv --log-file gpurun_out/linv_launches.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu6b.log 2>&1
echo done
