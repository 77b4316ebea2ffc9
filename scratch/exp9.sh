set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CMD="python bench.py --config 1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0"
cp paper_1707_05647_b200/csrc/ss_screen.cu /tmp/ss_screen_new.cu
cp scratch/ss_screen_head.cu paper_1707_05647_b200/csrc/ss_screen.cu
SS_ONLY=ss_screen.cu python paper_1707_05647_b200/build_native.py > /dev/null 2>&1
SS_STREAMS=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l9_head.csv $CMD > /dev/null 2>&1
cp /tmp/ss_screen_new.cu paper_1707_05647_b200/csrc/ss_screen.cu
SS_ONLY=ss_screen.cu python paper_1707_05647_b200/build_native.py > /dev/null 2>&1
SS_STREAMS=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l9_new.csv $CMD > /dev/null 2>&1
SS_STREAMS=1 SS_LIST_MODE=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l9_new_large.csv $CMD > /dev/null 2>&1
echo done
