#!/bin/bash
# Round evidence on one B200, in two phases (the bench lines quote the launch
# lists' DRAM / L2 / instruction counts, so the lists come first):
#   bash tools/evidence.sh TAG lists   ncu launch lists of configs 0-4 and
#                                      ncu --set full of stage 1 / rings / build
#   (here: python tools/launches.py ... --k3 configN -> profiles/r2/k3_traffic.json)
#   bash tools/evidence.sh TAG bench   bench lines for configs 0-4 (default =
#                                      config 4) and the reference arm
# Outputs under gpurun_out/ev_<tag>/.
TAG=${1:-r2}
PHASE=${2:-bench}
O=gpurun_out/ev_$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
if [ "$PHASE" = "lists" ]; then
  for c in 4 1 2 3 0; do
    CMD="python bench.py --config $c --steps 2 --warmup 1 --profile --graph 0"
    timeout 900 $CMD > /dev/null 2>&1 || { echo "plain run failed: config $c"; continue; }
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum \
        --clock-control none --csv --log-file $O/launches_config$c.csv $CMD > /dev/null 2>&1
  done
  for c in 4 1; do
    CMD="python bench.py --config $c --steps 2 --warmup 1 --profile --graph 0"
    N=8; [ $c = 1 ] && N=1
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ladder_stage1_coarse" -s 2 -c 1 \
        -o $O/ncu_stage1_c$c $CMD > /dev/null 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ladder_rings" -s 0 -c $N \
        -o $O/ncu_rings_c$c $CMD > /dev/null 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:band_kernel" -s 0 -c 1 \
        -o $O/ncu_build_c$c $CMD > /dev/null 2>&1
  done
else
  timeout 900 python bench.py > $O/bench_config4.json 2> $O/bench_config4.err
  for c in 0 1 2 3; do
    timeout 900 python bench.py --config $c > $O/bench_config$c.json 2> $O/bench_config$c.err
  done
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_config4.json 2> $O/bench_reference.err
fi
ls -la $O
