python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_leafinv -s 0 -c 1 -o gpurun_out/leafinv_v2 -f python scripts/factor_once.py cfg5 > gpurun_out/ncu_inv.log 2>&1
echo done
