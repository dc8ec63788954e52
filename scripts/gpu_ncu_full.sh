# ncu --set full captures of the largest launch of each top kernel of one
# config-5 factor (run under gpurun, one GPU).  Args: tag, then NAME:SKIP
# pairs (SKIP = index of the launch among that kernel's launches).
tag=$1; shift
for ks in "$@"; do
  k=${ks%%:*}; s=${ks##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" \
    --launch-skip $s -c 1 -o gpurun_out/ncu_${tag}_${k} -f \
    python scripts/factor_once.py cfg5 1 > gpurun_out/ncu_${tag}_${k}.log 2>&1
  echo "$k rc=$?"
done
