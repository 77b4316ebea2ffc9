#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over one small
# screen per config (tools/sanitize_case.py); logs -> gpurun_out/sanitize_<tag>_*.log
TAG=${1:-r2}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for c in "0" "1 768"; do
    name=$(echo "$c" | tr ' ' '_')
    timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
        python tools/sanitize_case.py $c > gpurun_out/sanitize_${TAG}_${tool}_c${name}.log 2>&1
    echo "$tool config $c rc=$?" | tee -a gpurun_out/sanitize_${TAG}_summary.txt
    tail -3 gpurun_out/sanitize_${TAG}_${tool}_c${name}.log
  done
done
