python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trunc_big -s 500 -c 2 -o gpurun_out/prof_tbig python scripts/factor_once.py cfg5 > gpurun_out/ncu4a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_leafinv -s 345 -c 1 -o gpurun_out/prof_linv python scripts/factor_once.py cfg5 > gpurun_out/ncu4b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trunc_warp -s 150 -c 1 -o gpurun_out/prof_twarp python scripts/factor_once.py cfg5 > gpurun_out/ncu4c.log 2>&1
echo done
