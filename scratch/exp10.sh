set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CMD="python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0"
SS_STREAMS=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l10_new.csv $CMD > /dev/null 2>&1
rm -f gpurun_out/variants.txt
VARIANTS="gc8:" CONFIGS="1 4 3" bash scratch/variants.sh
