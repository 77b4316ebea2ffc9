# usage: VARIANTS="name:ENV=1 ENV2=2;name2:..." CONFIGS="1 4" bash scratch/envvariants.sh
set -u
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%:*}; envs=${v#*:}
  for c in ${CONFIGS:-1 4}; do
    env $envs python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/env_${name}_c$c.log 2>&1
    grep '^{' gpurun_out/env_${name}_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$name', 'c$c', 'ms %.3f'%d['ms_per_step'], 'K3 %.3f'%r['screen_ms_per_step'], d['clocks'].get('sm_mhz'))" >> gpurun_out/envvariants.txt
  done
done
cat gpurun_out/envvariants.txt
