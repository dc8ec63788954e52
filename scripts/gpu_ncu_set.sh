# ncu --set full captures of the current top kernels (cfg5 factor): one launch each
for spec in "k_hmatB_sm 127" "k_leafgemm_tc 3" "k_leafinv_v2 0" "k_lu_panel_blk 0"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/v12_$1 -f python scripts/factor_once.py cfg5 > gpurun_out/ncu_$1.log 2>&1 < /dev/null
done
echo done > gpurun_out/ncuset_done
