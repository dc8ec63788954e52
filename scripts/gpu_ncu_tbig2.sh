python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_trunc_big -s 250 -c 1 -o gpurun_out/tbig_mid -f python scripts/factor_once.py cfg5 > gpurun_out/ncu_tbig.log 2>&1
echo done
