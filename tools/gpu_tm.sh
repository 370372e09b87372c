#!/bin/bash
# TMEM engine check: device product self-test, config-1 gates vs the oracle
# digests, then config-1 bench A/B (plain runs, no profiler).
#   gpurun --timeout 1500 -- 'bash tools/gpu_tm.sh TAG [bench args...]'
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fft_selftest.py tests/test_gpu_gates.py -q -p no:cacheprovider \
    -k "tmem or selftest" -x > gpurun_out/pytest_tm_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_tm_$TAG.log
for V in "$@"; do
  NAME=${V%%:*}; ARGS=${V#*:}
  timeout 600 python bench.py --no-net --steps 5 --warmup 3 $ARGS > gpurun_out/ab_${TAG}_$NAME.log 2>&1
  echo "exit $?" >> gpurun_out/ab_${TAG}_$NAME.log
done
exit 0
