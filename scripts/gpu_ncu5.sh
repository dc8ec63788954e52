nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 250 > gpurun_out/clk.csv &
SMI=$!
REPS=6 python scripts/time_configs.py cfg5 > gpurun_out/t5.log 2>&1
kill $SMI
python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_leafinv -s 345 -c 1 -o gpurun_out/prof_linv2 python scripts/factor_once.py cfg5 > gpurun_out/ncu5.log 2>&1
echo done
