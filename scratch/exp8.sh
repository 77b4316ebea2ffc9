set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_screen.py -x -q > gpurun_out/exp8_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/exp8_tests.log
VARIANTS="exact_rings:;fast_rings:-DRINGS_FAST_CM=1;exact_both:-DSTAGE1_FAST_CM=0;minb2:-DRINGS_MINB=2" bash scratch/exp6.sh
