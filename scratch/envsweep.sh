#!/bin/bash
# for each "NAME=VAL" setting in $SWEEP (space separated), run bench --config $C and print K3/step ms
C=${C:-4}
mkdir -p gpurun_out
for kv in $SWEEP; do
  env $kv timeout 400 python bench.py --config $C --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/sw.json 2> gpurun_out/sw.err
  python - "$kv" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/sw.json").read().strip().splitlines()[-1])
print(f"{sys.argv[1]:>32s}  K3 {d['roofline']['screen_ms_per_step']:.3f} ms  step {d['ms_per_step']:.3f} ms  {d['value']/1e9:.2f} G/s {d['clocks']['reasons']}")
PY
done
