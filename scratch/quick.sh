#!/bin/bash
# gpu tests + benches for the given configs (default 1) + fused profile of config 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log | grep -v "^\.\.\." | tail -15
for c in ${CONFIGS:-1}; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bf_c$c.json 2> gpurun_out/bf_c$c.err; echo bench $c rc=$?; done
[ -n "$PROF" ] && bash scratch/prof_fused.sh 1 $PROF
true
