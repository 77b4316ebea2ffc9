#!/bin/bash
# bench lines for all five BASELINE configs (single GPU) -> gpurun_out/bench_config*.json
mkdir -p gpurun_out
for c in 0 1 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_config$c.log 2>&1
  echo "config $c rc=$?"
  grep '^{' gpurun_out/bench_config$c.log | tail -1 > gpurun_out/bench_config$c.json
done
