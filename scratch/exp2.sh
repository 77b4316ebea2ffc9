set -u
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/exp2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/exp2_tests.log
VARIANTS="${VARIANTS:-base:;minb4:-DRINGS_MINB=4;g256:-DRINGS_GROUP=256}" CONFIGS="${CONFIGS:-1 4 3}" bash scratch/variants.sh
