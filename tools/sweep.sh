#!/bin/bash
# Build-flag sweep on the GPU box: for each variant (nvcc -D flags for
# ss_ladder_screen.cu) rebuild and run the bench (no CPU legs, no e2e) on the
# given configs; one JSON summary line per (variant, config) in
# gpurun_out/sweep_<tag>.txt.  usage: bash tools/sweep.sh TAG "CONFIGS" "VARIANT1" "VARIANT2" ...
TAG=$1; shift
CONFIGS=$1; shift
OUT=gpurun_out/sweep_${TAG}.txt
mkdir -p gpurun_out
for v in "$@"; do
  SS_EXTRA_NVCC="$v" SS_ONLY=ss_ladder_screen.cu python -c "from paper_1707_05647_b200 import build_native; build_native.build()" \
    || { echo "build failed: $v" >> $OUT; continue; }
  for c in $CONFIGS; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2> /tmp/sweep.err | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(json.dumps({'variant': '$v', 'config': $c, 'ms_per_step': round(d['ms_per_step'],4), 'k3_ms': round(r['k3_ms_per_step'],4), 'value_G': round(d['value']/1e9,2), 'clocks': d['clocks']['sm_mhz']}))" >> $OUT \
      || { echo "run failed: $v config $c" >> $OUT; tail -3 /tmp/sweep.err >> $OUT; }
  done
done
# restore the default build
SS_ONLY=ss_ladder_screen.cu python -c "from paper_1707_05647_b200 import build_native; build_native.build()"
cat $OUT
