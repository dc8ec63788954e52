# ncu --set full captures of chosen launches of one config-5 factor (run under
# gpurun, one GPU).  Args: tag, then REGEX@SKIP pairs (SKIP = index of the
# launch among the launches whose demangled name matches REGEX).
tag=$1; shift
for ks in "$@"; do
  k=${ks%%@*}; s=${ks##*@}
  f=$(echo "$k" | tr -c 'A-Za-z0-9_\n' '_')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$k" --launch-skip $s -c 1 -o gpurun_out/ncu_${tag}_${f}_$s -f \
    python scripts/factor_once.py cfg5 1 > gpurun_out/ncu_${tag}_${f}_$s.log 2>&1
  echo "$k@$s rc=$?"
done
