#!/bin/bash
# The sanitizer substitute: rebuild with -DSS_DEBUG (SS_CHECK bounds checks
# trap on violation), run the GPU parity suite on it, restore the normal build.
mkdir -p gpurun_out
SS_EXTRA_NVCC="-DSS_DEBUG" python -c "from paper_1707_05647_b200 import build_native; build_native.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/debug_check.log
rc=$?
python -c "from paper_1707_05647_b200 import build_native; build_native.build()"
cat gpurun_out/debug_check.log
exit $rc
