# the round's closing measurement pass (run under gpurun): tests, smoke, bench
# lines, launch list + per-level times, solve launch list
set -x
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/tgpu.log 2>&1; echo "exit $?" >> gpurun_out/tgpu.log
tail -n 3 gpurun_out/tgpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -n 2
python bench.py > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err
python bench.py --impl reference > gpurun_out/r02_bench_ref_cfg5.json 2> gpurun_out/r02_bench_ref_cfg5.err
bash scripts/gpu_profile.sh r02h
python scripts/solve_once.py cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py cfg5 > gpurun_out/solve_ncu.log 2>&1
bash scripts/gpu_ncu_full.sh r02h "k_leafinv_tri@0"
for f in gpurun_out/ncu_r02h_k_leafinv_tri_0.ncu-rep; do python scripts/ncu_summary.py $f 14 > ${f%.ncu-rep}.txt 2>&1; done
rm -f gpurun_out/ncu_r02h_*.ncu-rep
