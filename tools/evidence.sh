#!/bin/bash
# Round evidence on one B200: bench lines for configs 0-4 (default = config 4),
# the reference arm, ncu launch lists per config, ncu --set full of the two
# dominant kernels at configs 4 and 1.  Outputs under gpurun_out/ev_<tag>/.
TAG=${1:-r2}
O=gpurun_out/ev_$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench_config4.json 2> $O/bench_config4.err
for c in 0 1 2 3; do
  timeout 900 python bench.py --config $c > $O/bench_config$c.json 2> $O/bench_config$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_config4.json 2> $O/bench_reference.err
for c in 4 1 2 3 0; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --profile --graph 0"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
      --clock-control none --csv --log-file $O/launches_config$c.csv $CMD > /dev/null 2>&1
done
for c in 4 1; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --profile --graph 0"
  S=5; [ $c = 1 ] && S=2
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ladder_stage1_coarse" -s $S -c 1 \
      -o $O/ncu_stage1_c$c $CMD > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ladder_rings" -s $S -c 1 \
      -o $O/ncu_rings_c$c $CMD > /dev/null 2>&1
done
ls -la $O
