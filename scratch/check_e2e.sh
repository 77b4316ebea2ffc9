mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ce_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ce_tests.log
for c in ${CONFIGS:-1 3 0}; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ce_b$c.log 2>&1
grep '^{' gpurun_out/ce_b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; e=d['e2e']; print('c$c', 'ms %.3f'%d['ms_per_step'], 'K3 %.3f'%r['screen_ms_per_step'], 'e2e_ms', [round(x,3) for x in e['ms_min_median_max']], 'launches', d['gpu_launches'])"
done
python scratch/e2e_prof.py 1 > gpurun_out/e2e_prof.log 2>&1
