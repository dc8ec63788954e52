# ncu --set full captures of the largest launch of every top kernel of one
# config-5 factor + text summaries (run under gpurun; outputs in gpurun_out/).
# The REGEX@SKIP picks come from the launch list (scripts/gpu_profile.sh):
# SKIP = index of the kernel's longest launch among its launches.
tag=${1:-r02}
bash scripts/gpu_ncu_full.sh $tag "k_trunc_warp@183" "k_trunc_big<\(int\)256>@131" "k_trunc_big<\(int\)512>@17" "k_trunc_pair@10" \
  "k_hmatB_tc@61" "k_hmatA_tcw@30" "k_leafgemm_tc@1" "k_leafinv_bgj@0" "k_gp_tc@93" "k_leaflr@14" \
  "k_schur_leaf@0" "k_lu_panel_reg@0" "k_trunc_classify@59" "k_trunc_big<\(int\)512>@540"
for f in gpurun_out/ncu_${tag}_*.ncu-rep; do python scripts/ncu_summary.py $f 14 > ${f%.ncu-rep}.txt 2>&1; done
rm -f gpurun_out/ncu_${tag}_*.ncu-rep   # the text summaries are what profiles/ keeps (gpurun_out/ is capped at 64 MiB)
ls -la gpurun_out/ncu_${tag}_*.txt
