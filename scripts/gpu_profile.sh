# launch list of one config-5 factor (ncu, serialised, cold) + per-level host
# timing of a warm factor (run under gpurun; outputs in gpurun_out/)
set -x
tag=${1:-r02}
ACR_DEBUG=1 python scripts/factor_once.py cfg5 3 > gpurun_out/levels_$tag.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv python scripts/factor_once.py cfg5 1 > gpurun_out/ncu_$tag.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$tag.csv -v > gpurun_out/launches_${tag}_summary.txt
tail -5 gpurun_out/ncu_$tag.log
