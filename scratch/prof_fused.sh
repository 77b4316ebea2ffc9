#!/bin/bash
# fused ladder: launch list + ncu full of both fused kernels (config ${1:-1})
C=${1:-1}; TAG=${2:-r1o}
mkdir -p gpurun_out
CMD="python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --graph 0"
$CMD > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_config$C.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:ladder_stage1 -s 1 -c 1 -o gpurun_out/prof_s1_${TAG}_c$C $CMD > gpurun_out/ncu_s1.log 2>&1
echo s1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:ladder_rings -s 1 -c 1 -o gpurun_out/prof_rk_${TAG}_c$C $CMD > gpurun_out/ncu_rk.log 2>&1
echo rk rc=$?
