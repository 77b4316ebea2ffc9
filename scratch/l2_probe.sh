# stage1 L2/DRAM behaviour on config 4 under TMA promotion / strip variants
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_hit.sum,lts__t_sectors_op_read_lookup_miss.sum
CMD="python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0"
python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_probe.log 2>&1 || exit 1
for v in "3 x" "0 x" "3 64" "3 16"; do
  set -- $v
  if [ "$2" = x ]; then unset SS_STRIP; else export SS_STRIP=$2; fi
  SS_TMA_PROMO=$1 ncu --metrics $M --clock-control none -k regex:stage1 -c 33 --csv --log-file gpurun_out/probe_p$1_s$2.csv $CMD > /dev/null 2>&1
  echo "variant $v rc=$?"
done
