python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_trunc --csv --log-file gpurun_out/trunc_dram.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu_traffic.log 2>&1
echo done
