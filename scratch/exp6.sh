set -u
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
cp paper_1707_05647_b200/csrc/ss_screen.cu /tmp/ss_screen_new.cu
cp scratch/ss_screen_head.cu paper_1707_05647_b200/csrc/ss_screen.cu
VARIANTS="head:" CONFIGS="${CONFIGS:-1 4 3}" bash scratch/variants.sh > /dev/null
cp /tmp/ss_screen_new.cu paper_1707_05647_b200/csrc/ss_screen.cu
VARIANTS="${VARIANTS}" CONFIGS="${CONFIGS:-1 4 3}" bash scratch/variants.sh
