set -u
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
VARIANTS="b512:;b64:-DLIST_BLOCK_MAX=64;b32:-DLIST_BLOCK_MAX=32" CONFIGS="1 4 3" bash scratch/variants.sh
SS_ONLY=ss_screen.cu python paper_1707_05647_b200/build_native.py > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_exp3_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 > /dev/null 2>&1
echo done
