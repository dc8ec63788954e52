python scripts/factor_once.py cfg2 > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trunc -s 120 -c 2 -o gpurun_out/prof_trunc_v0 python scripts/factor_once.py cfg2 > gpurun_out/ncu_full_v0.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full_v0.log
