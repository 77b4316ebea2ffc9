# quick check: parity tests + short benches (no cpu baseline / e2e)
mkdir -p gpurun_out
rm -f gpurun_out/quick.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick.txt
tail -2 gpurun_out/quick_tests.log >> gpurun_out/quick.txt
for c in ${CONFIGS:-1 4 3}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick_c$c.log 2>&1
  grep '^{' gpurun_out/quick_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c$c', 'ms %.3f'%d['ms_per_step'], 'K3 %.3f'%r['screen_ms_per_step'], 'G/s %.1f'%(d['value']/1e9), 'frac %.3f'%r['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" >> gpurun_out/quick.txt
done
cat gpurun_out/quick.txt
