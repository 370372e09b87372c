#!/bin/bash
# The checked build (libshe.so with -DSHE_CHECKED: device bounds checks on the
# default path, csrc/dcheck.cuh; compute-sanitizer is closed on this pool):
# tools/build_variant.sh varbuild/checked.so -DSHE_CHECKED, swapped in for the
# small all-kernel workload and the gate-level GPU tests.
#   gpurun --timeout 1800 -- 'bash tools/gpu_checked.sh TAG'
set -u
TAG=${1:-chk}
mkdir -p gpurun_out
L=paper_1906_00148_b200/libshe.so
cp $L /tmp/libshe_default.so
cp varbuild/checked.so $L && touch $L
timeout 600 python tools/sanitize_small.py > gpurun_out/checked_small_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/checked_small_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_gates.py tests/test_gpu_fft_selftest.py -q -p no:cacheprovider \
    > gpurun_out/checked_pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/checked_pytest_$TAG.log
cp /tmp/libshe_default.so $L
exit 0
