set -u
mkdir -p gpurun_out
python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 4; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 0 1 2 3 4; do
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_config$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 > /dev/null 2>&1
done
echo done
