set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputest_a.log
timeout 900 python bench.py > gpurun_out/bench_c4_a.json 2> gpurun_out/bench_c4_a.err
tail -5 gpurun_out/bench_c4_a.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_a.json 2> gpurun_out/bench_ref_a.err
tail -3 gpurun_out/bench_ref_a.err
timeout 900 bash tools/profile.sh r2a 4 ladder_rings_kernel 3 1 > gpurun_out/prof_a.log 2>&1
cat gpurun_out/prof_a.log
