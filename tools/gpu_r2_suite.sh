#!/bin/bash
# Round 2: full GPU suite, then config-1 A/B of the engine options given as
# "name:args" pairs (plain bench runs, --no-net).
#   gpurun --timeout 2400 -- 'bash tools/gpu_r2_suite.sh TAG "v2:" "v3:--fft-variant 3" ...'
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
for V in "$@" "ksimma:--ks-kernel imma" "kscuda:--ks-kernel cuda"; do
  NAME=${V%%:*}; ARGS=${V#*:}
  timeout 600 python bench.py --no-net --steps 5 --warmup 3 $ARGS > gpurun_out/ab_${TAG}_$NAME.log 2>&1
  echo "exit $?" >> gpurun_out/ab_${TAG}_$NAME.log
done
exit 0
