set -x
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 python scripts/sanitize_case.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -n 6 gpurun_out/sanitize_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 7 python scripts/race_case.py 64 8 > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"
tail -n 6 gpurun_out/sanitize_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 7 python scripts/race_case.py 64 8 > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"
tail -n 4 gpurun_out/sanitize_synccheck.log
