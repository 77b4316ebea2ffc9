#!/bin/bash
# Round evidence: bench lines of all configs (+ reference arm), ncu launch lists (+DRAM bytes) per config.
TAG=${1:-r1u}
mkdir -p gpurun_out/$TAG
for c in 1 0 2 3 4; do
  timeout 400 python bench.py --config $c > gpurun_out/$TAG/bench_config$c.json 2> gpurun_out/$TAG/bench_config$c.err; echo bench $c rc=$?
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_reference_config1.json 2> gpurun_out/$TAG/bench_ref.err; echo ref rc=$?
for c in 1 0 2 3 4; do
  ST=2; [ $c = 4 ] && ST=1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/$TAG/launches_${TAG}_config$c.csv python bench.py --config $c --steps $ST --warmup 1 --no-cpu-baseline --no-e2e --graph 0 > gpurun_out/$TAG/ncu_c$c.log 2>&1
  echo launches $c rc=$?
done
