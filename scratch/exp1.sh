set -u
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt gpurun_out/envvariants.txt
VARIANTS="g128:-DRINGS_GROUP=128;g64:-DRINGS_GROUP=64;g32:-DRINGS_GROUP=32;g32c16:-DRINGS_GROUP=32 -DRINGS_COUNTERS=16" CONFIGS="1 4 3" bash scratch/variants.sh
SS_ONLY=ss_screen.cu SS_EXTRA_NVCC="-DRINGS_GROUP=32" python paper_1707_05647_b200/build_native.py > /dev/null 2>&1
VARIANTS="s1:SS_STREAMS=1;s2:SS_STREAMS=2;s4:SS_STREAMS=4;p12:SS_STRIP_PLANES=12;p6:SS_STRIP_PLANES=6" CONFIGS="1 4" bash scratch/envvariants.sh
