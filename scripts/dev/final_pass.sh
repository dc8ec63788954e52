set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err
python bench.py --impl reference > gpurun_out/r02_bench_ref_cfg5.json 2> gpurun_out/r02_bench_ref_cfg5.err
bash scripts/gpu_profile.sh r02h
bash scripts/gpu_ncu_full.sh r02h "k_gp_tc@93" "k_trunc_big<\(int\)512>@17" "k_hmatB_tc@61"
for f in gpurun_out/ncu_r02h_*.ncu-rep; do python scripts/ncu_summary.py $f 14 > ${f%.ncu-rep}.txt 2>&1; done
rm -f gpurun_out/ncu_r02h_*.ncu-rep
python scripts/solve_once.py cfg5
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py cfg5 > gpurun_out/solve_ncu.log 2>&1
