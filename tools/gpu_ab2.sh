#!/bin/bash
# Round 2 A/B: GPU tests, then config-1 bench for each FFT shape / batch size
# given as "name:args" pairs (bench.py --no-net, plain runs, no profiler).
#   gpurun --timeout 1800 -- 'bash tools/gpu_ab2.sh TAG [tests] "fft4:" "fft3:--fft-lanes 3" ...'
set -u
TAG=$1; shift
mkdir -p gpurun_out
if [ "${1:-}" = "tests" ]; then
  shift
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
fi
for V in "$@"; do
  NAME=${V%%:*}; ARGS=${V#*:}
  timeout 600 python bench.py --no-net --steps 5 --warmup 3 $ARGS > gpurun_out/ab_${TAG}_$NAME.log 2>&1
  echo "exit $?" >> gpurun_out/ab_${TAG}_$NAME.log
done
exit 0
