mkdir -p gpurun_out/ab2
SS_BUILD_KINDS=4 timeout 300 python tools/build_ab.py > gpurun_out/ab2/k4.json 2> /dev/null; echo rc=$?
timeout 300 python tools/build_ab.py > gpurun_out/ab2/def.json 2> /dev/null; echo rc=$?
SS_BUILD_KINDS=2 timeout 300 python tools/build_ab.py > gpurun_out/ab2/k2.json 2> /dev/null; echo rc=$?
SS_BAND_ROWS=15 SS_BUILD_KINDS=4 timeout 300 python tools/build_ab.py --cases odd --reps 2 > gpurun_out/ab2/k4_15.json 2>/dev/null
SS_BAND_ROWS=15 SS_BUILD_KINDS=2 timeout 300 python tools/build_ab.py --cases odd --reps 2 > gpurun_out/ab2/k2_15.json 2>/dev/null
timeout 600 python -m pytest tests/test_gpu_tables.py -x -q > gpurun_out/ab2/tables.log 2>&1; echo tables rc=$?
