set -u
mkdir -p gpurun_out
TAG=${TAG:-r1m}
for c in 1 4; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 0 1 2 3 4; do
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_${TAG}_config$c.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 > /dev/null 2>&1
done
CMD="python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0"
ncu --set full --clock-control none --import-source on -k regex:"stage1|rings_kernel" -s 8 -c 2 -o gpurun_out/prof_${TAG}_c1 $CMD > gpurun_out/ncu_full_${TAG}_c1.log 2>&1
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0"
ncu --set full --clock-control none --import-source on -k regex:"stage1|rings_kernel" -s 40 -c 2 -o gpurun_out/prof_${TAG}_c4 $CMD > gpurun_out/ncu_full_${TAG}_c4.log 2>&1
echo done
