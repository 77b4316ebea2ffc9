#!/bin/bash
# Usage (on the GPU box): bash tools/profile.sh <tag> <config> [kernel-regex] [skip] [count]
# 1) plain bench run (must exit 0), 2) ncu launch list (time, DRAM bytes, warp
# instructions per launch), 3) ncu --set full on the chosen kernel.
set -u
TAG=${1:-r2}
CFG=${2:-4}
KRE=${3:-ladder_rings_kernel}
SKIP=${4:-0}
CNT=${5:-1}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --profile --graph 0"
$CMD > gpurun_out/plain_${TAG}_c$CFG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c$CFG.csv $CMD > gpurun_out/ncu_launch_${TAG}_c$CFG.log 2>&1
echo "launch list rc=$?"
if [ "$CNT" != "0" ]; then
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s $SKIP -c $CNT \
    -o gpurun_out/prof_${TAG}_c$CFG $CMD > gpurun_out/ncu_full_${TAG}_c$CFG.log 2>&1
echo "full rc=$?"
fi
