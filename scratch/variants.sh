# usage: VARIANTS="name:flags;name2:flags2" CONFIGS="1 4" bash scratch/variants.sh
set -u
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  SS_ONLY=ss_screen.cu SS_EXTRA_NVCC="$flags" python paper_1707_05647_b200/build_native.py > gpurun_out/build_$name.log 2>&1 || { echo "build $name failed"; continue; }
  for c in ${CONFIGS:-1 4}; do
    python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_${name}_c$c.log 2>&1
    grep '^{' gpurun_out/var_${name}_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$name', 'c$c', 'ms %.3f'%d['ms_per_step'], 'K3 %.3f'%r['screen_ms_per_step'], d['clocks'].get('sm_mhz'))" >> gpurun_out/variants.txt
  done
  if [ -n "${NCU:-}" ]; then
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"${NCU}" --csv --log-file gpurun_out/var_${name}_ncu.csv python bench.py --config ${NCU_CONFIG:-4} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 > /dev/null 2>&1
  fi
done
cat gpurun_out/variants.txt
