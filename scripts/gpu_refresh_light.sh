# bench lines (both arms) and the launch list (cfg5), no full captures
V=${V:-v13}
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$V.json 2>> gpurun_out/bench_$V.err
python scripts/factor_once.py cfg5 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_cfg5_$V.csv python scripts/factor_once.py cfg5 > gpurun_out/ncu_l.log 2>&1 < /dev/null
echo done > gpurun_out/refresh_done
