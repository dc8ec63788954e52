# ncu --set full of the solve's level-0 HODLR x panel launches (phase B and A)
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_hmatB_sm -s 1 -c 1 -o gpurun_out/solve_hmatB -f python scripts/solve_once.py > gpurun_out/ncu_sB.log 2>&1 < /dev/null
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_hmatA -s 0 -c 1 -o gpurun_out/solve_hmatA -f python scripts/solve_once.py > gpurun_out/ncu_sA.log 2>&1 < /dev/null
echo done
