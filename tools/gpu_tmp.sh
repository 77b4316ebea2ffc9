mkdir -p gpurun_out/ab4
timeout 300 python tools/build_ab.py > gpurun_out/ab4/def.json 2> /dev/null; echo rc=$?
SS_BUILD_KINDS=2 timeout 300 python tools/build_ab.py --cases big --reps 5 > gpurun_out/ab4/k2.json 2> /dev/null; echo rc=$?
for rb in 15 31 63; do SS_BAND_ROWS=$rb timeout 300 python tools/build_ab.py --cases odd,small --reps 2 > gpurun_out/ab4/def_$rb.json 2>/dev/null; done
timeout 600 python -m pytest tests/test_gpu_tables.py -x -q > gpurun_out/ab4/tables.log 2>&1; echo tables rc=$?
