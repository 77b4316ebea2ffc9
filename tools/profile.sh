#!/bin/bash
# Usage (on the GPU box): bash tools/profile.sh <tag> [kernel-regex] [skip] [count]
# 1) plain bench run (must exit 0), 2) ncu launch list, 3) ncu --set full on the chosen kernel.
set -u
TAG=${1:-r1}
KRE=${2:-ring_kernel|stage1_kernel}
SKIP=${3:-20}
CNT=${4:-4}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --graph 0"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s $SKIP -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile rc=$?"
