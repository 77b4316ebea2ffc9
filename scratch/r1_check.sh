#!/bin/bash
# GPU tests + bench lines for all configs on the current tree
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
for c in 1 0 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_config$c.log 2>&1
  echo "config $c rc=$?"
  grep '^{' gpurun_out/bench_config$c.log | tail -1 > gpurun_out/bench_config$c.json
done
