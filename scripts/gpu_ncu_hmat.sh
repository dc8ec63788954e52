python scripts/solve_once.py > gpurun_out/solve_plain.log 2>&1 && \
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_hmatB -c 1 -o gpurun_out/hmatB_solve -f python scripts/solve_once.py > gpurun_out/ncu_hmat.log 2>&1
echo done
