#!/bin/bash
# Build-flag variants on the GPU box: for each "name|flags" in $VARIANTS, rebuild
# with SS_EXTRA_NVCC=flags and run the bench on $CONFIGS; prints K3 ms and step ms.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%|*}; flags=${v#*|}
  SS_EXTRA_NVCC="$flags" python -m paper_1707_05647_b200.build_native > /dev/null 2> gpurun_out/build_$name.err || { echo "$name build failed"; continue; }
  for c in ${CONFIGS:-1}; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/var_${name}_c$c.json 2> gpurun_out/var_${name}_c$c.err
    python - "$name" "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/var_{sys.argv[1]}_c{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:>14s} c{sys.argv[2]}  K3 {d['roofline']['screen_ms_per_step']:.4f} ms  step {d['ms_per_step']:.4f} ms  {d['value']/1e9:.2f} G/s")
PY
  done
done
