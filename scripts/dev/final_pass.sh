set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err
python bench.py --impl reference > gpurun_out/r02_bench_ref_cfg5.json 2> gpurun_out/r02_bench_ref_cfg5.err
bash scripts/gpu_profile.sh r02h
bash scripts/gpu_ncu_round.sh r02h
bash scripts/gpu_traffic.sh
python scripts/trunc_phases.py > gpurun_out/phases_r02h.txt 2>&1
python scripts/solve_once.py cfg5
